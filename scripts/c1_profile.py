import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2405_05155_b200 import configs, relaxation
from paper_2405_05155_b200.kernels import kernel_spec
c1 = configs.c1_relax(seed=0)
spec = kernel_spec("laguerre-gauss", c1["h"], 2)
rl = relaxation.PeriodicRelaxer(c1["pos"], spec, c1["box"], c1["dp"], step_scale=c1["step_scale"])
rl.run(3, graph=False)
torch.cuda.synchronize()
rl.run(2, graph=False)
torch.cuda.synchronize()
