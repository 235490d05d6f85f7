"""Large-size check of the WC engine (GPU box): TGV-3D at n_side^3 with the
2h kernel, where the ELL pass list has more than 2^31 entries
(384^3 x 80 = 4.5e9): a few steps, mass conservation, finite fields, time.
    python scripts/large_check.py [n_side] [kernel] [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver,
                                                FluidState)

    n_side = int(sys.argv[1]) if len(sys.argv) > 1 else 384
    kernel = sys.argv[2] if len(sys.argv) > 2 else "2h"
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    cfg = configs.c5_tgv3d(kernel=kernel, n_side=n_side)
    n = cfg["pos"].shape[0]
    t0 = time.time()
    s = EulerianSolver(cfg["pos"], n, FluidState(cfg["vol"], cfg["rho"], cfg["mom"], None, n),
                       EosParams(WEAKLY_COMPRESSIBLE, rho0=cfg["rho0"], c_art=cfg["c_art"]),
                       cfg["spec"], None, cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
    setup = time.time() - t0
    m0 = float(np.sum(cfg["vol"] * cfg["rho"]))
    s.advance(2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.advance(steps)
    e1.record()
    torch.cuda.synchronize()
    st = s.state
    m1 = float(np.sum(st.vol * st.rho))
    print(json.dumps({"n_side": n_side, "n": n, "kernel": kernel, "width": s.width,
                      "pass_list_entries": int(s.width) * n,
                      "pairs": int(s.cnt.sum().item()), "setup_s": setup,
                      "ms_per_step": e0.elapsed_time(e1) / steps,
                      "finite": bool(np.isfinite(st.rho).all() and np.isfinite(st.mom).all()),
                      "mass_rel_drift": abs(m1 - m0) / m0,
                      "gpu_mem_gb": torch.cuda.max_memory_allocated() / 1e9}))


if __name__ == "__main__":
    main()
