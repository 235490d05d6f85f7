import sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_2405_05155_b200 import configs
from paper_2405_05155_b200.eulerian import WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver, FluidState
torch.zeros(1, device='cuda')
cfg = configs.c5_tgv3d(kernel="1.6h", n_side=256)
n = cfg["pos"].shape[0]
t0 = time.perf_counter()
s = EulerianSolver(cfg["pos"], n, FluidState(cfg["vol"], cfg["rho"], cfg["mom"], None, n),
                   EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0), cfg["spec"], None,
                   cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
torch.cuda.synchronize()
print("setup_s", time.perf_counter() - t0)
