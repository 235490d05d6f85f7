"""C2 TGV-2D (40k particles, 1.6h) WC steps for profiling (GPU box)."""
import sys; sys.path.insert(0, '/root/repo')
from paper_2405_05155_b200 import configs
from paper_2405_05155_b200.eulerian import WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver, FluidState
import torch
cfg = configs.c2_tgv2d(kernel="1.6h"); n = cfg["pos"].shape[0]
s = EulerianSolver(cfg["pos"], n, FluidState(cfg["vol"], cfg["rho"], cfg["mom"], None, n), EosParams(WEAKLY_COMPRESSIBLE, rho0=cfg["rho0"], c_art=cfg["c_art"]), cfg["spec"], None, cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
s.advance(4, graph=False); torch.cuda.synchronize()
