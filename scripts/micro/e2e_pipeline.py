"""Diagnostic of the e2e state-transfer pipeline (bench.py e2e_leg): the same
loop with the step removed (copies only) and with a fixed-dt step, C5 256^3."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2405_05155_b200 import configs  # noqa: E402
from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams,  # noqa: E402
                                            EulerianSolver, FluidState)

cfg = configs.c5_tgv3d(kernel="1.6h", n_side=256)
n = cfg["pos"].shape[0]
st = FluidState(cfg["vol"], cfg["rho"], cfg["mom"], None, n)
s = EulerianSolver(cfg["pos"], n, st, EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0),
                   cfg["spec"], None, cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
rho_in = torch.empty(n, dtype=torch.float64).pin_memory()
mom_in = torch.empty((n, 3), dtype=torch.float64).pin_memory()
rho_out = torch.empty(n, dtype=torch.float64).pin_memory()
mom_out = torch.empty((n, 3), dtype=torch.float64).pin_memory()
s.read_state(rho_in, mom_in)
torch.cuda.synchronize()
dt = s.compute_dt()
for mode in ("copies only", "step()", "step(dt)", "advance(1)"):
    last = []

    def one():
        s.load_state(rho_in, mom_in)
        s.prefetch_state(rho_in, mom_in)
        if mode == "step()":
            s.step()
        elif mode == "step(dt)":
            s.step(dt)
        elif mode == "advance(1)":
            s.advance(1)
        last[:] = [s.read_state(rho_out, mom_out, wait=False)]

    s.prefetch_state(rho_in, mom_in)
    for _ in range(2):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(8):
        one()
    torch.cuda.current_stream().wait_event(last[0])
    torch.cuda.current_stream().wait_event(s._io["prefetched"][2])
    e1.record()
    torch.cuda.synchronize()
    print(mode, "%.2f ms/step" % (e0.elapsed_time(e1) / 8), flush=True)
