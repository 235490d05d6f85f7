"""Long-run check of the C5 engine: TGV-3D at Re = 1600 to t = 10 on a
128^3 lattice with the truncated (1.6h) and standard (2h) Wendland kernels.
Records the volume-averaged kinetic energy E_k(t) = sum V rho |v|^2 / (2 sum V)
and mass conservation; prints one JSON object.  (GPU box; ~30 s.)"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(kernel, n_side, t_end, dt_out):
    import torch

    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver,
                                                FluidState)

    cfg = configs.c5_tgv3d(kernel=kernel, n_side=n_side)
    n = cfg["pos"].shape[0]
    s = EulerianSolver(cfg["pos"], n, FluidState(cfg["vol"], cfg["rho"], cfg["mom"], None, n),
                       EosParams(WEAKLY_COMPRESSIBLE, rho0=cfg["rho0"], c_art=cfg["c_art"]),
                       cfg["spec"], None, cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
    vol = cfg["vol"]

    def energy():
        st = s.state
        v2 = np.sum(st.mom**2, axis=1) / st.rho
        return float(0.5 * np.sum(vol * v2) / np.sum(vol)), float(np.sum(vol * st.rho))

    ts, es = [0.0], [energy()[0]]
    m0 = energy()[1]
    steps = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    while s.t < t_end - 1e-12:
        target = min(s.t + dt_out, t_end)
        while s.t < target - 1e-12:
            s.advance(50)          # CFL steps, CUDA-graph replay
            steps += 50
        ts.append(s.t)
        es.append(energy()[0])
    wall = time.perf_counter() - t0
    return {"kernel": kernel, "t": ts, "ek": es, "steps": steps, "wall_s": wall,
            "mass_rel_drift": abs(energy()[1] - m0) / m0, "pairs_per_particle": s.width}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-side", type=int, default=128)
    ap.add_argument("--t-end", type=float, default=10.0)
    ap.add_argument("--dt-out", type=float, default=0.5)
    a = ap.parse_args()
    legs = {k: run(k, a.n_side, a.t_end, a.dt_out) for k in ("1.6h", "2h")}
    tw, sw = legs["1.6h"], legs["2h"]
    diff = float(np.max(np.abs(np.interp(sw["t"], tw["t"], tw["ek"]) - np.asarray(sw["ek"]))) /
                 sw["ek"][0])
    print(json.dumps({"n_side": a.n_side, "re": 1600, "legs": legs,
                      "max_ek_diff_tw_vs_sw_rel_to_ek0": diff,
                      "alpha_wall": tw["wall_s"] / sw["wall_s"]}))


if __name__ == "__main__":
    main()
