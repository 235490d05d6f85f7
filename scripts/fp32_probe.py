"""Time the optional FP32 mode of the C5 stage engine (GPU box).

    python scripts/fp32_probe.py [--n-side 256] [--steps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-side", type=int, default=256)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--precision", default="fp32")
    args = ap.parse_args()
    import torch

    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver,
                                                FluidState)

    cfg = configs.c5_tgv3d(kernel="1.6h", n_side=args.n_side)
    n = cfg["pos"].shape[0]
    s = EulerianSolver(cfg["pos"], n, FluidState(cfg["vol"], cfg["rho"], cfg["mom"], None, n),
                       EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0), cfg["spec"], None,
                       cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"],
                       precision=args.precision)
    s.advance(2, graph=False)
    torch.cuda.synchronize()
    s.timer = []
    s.advance(args.steps, graph=False)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for _, a, b in s.timer]
    s.timer = None
    s.advance(4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.advance(20)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"precision": args.precision, "stage_ms": sum(ms) / len(ms),
                      "graph_ms_per_step": e0.elapsed_time(e1) / 20}))


if __name__ == "__main__":
    main()
