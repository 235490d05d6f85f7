"""Sweep launch variants of the WC stage kernel on one config (GPU box).

    python scripts/tune_wc.py [--n-side 192] [--kernel 1.6h]

Each variant runs in a fresh process (the variant switches are read once per
process): SPHB_WC_KERNEL (global|tiled), SPHB_WC_GROUP (lanes per particle),
SPHB_WC_MINB (min resident CTAs -> register cap).  Prints one JSON line per
variant with the mean stage time (CUDA events).
"""

import argparse
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(n_side, kernel, steps, precision="fp64"):
    sys.path.insert(0, REPO)
    import torch

    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver,
                                                FluidState)

    cfg = configs.c5_tgv3d(kernel=kernel, n_side=n_side)
    n = cfg["pos"].shape[0]
    st = FluidState(cfg["vol"], cfg["rho"], cfg["mom"], None, n)
    s = EulerianSolver(cfg["pos"], n, st, EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0),
                       cfg["spec"], None, cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"],
                       precision=precision)
    s.advance(3)
    torch.cuda.synchronize()
    if os.environ.get("SPHB_EXPERIMENT"):     # raw stage-1 launches into scratch
        out = torch.empty_like(s.S)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.params.reserved = int(os.environ["SPHB_EXPERIMENT"])
        e0.record()
        for _ in range(10):
            s._launch_stage_raw(1, s.S, s.S, s.M, out, None)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"experiment": s.params.reserved, "stage_ms": e0.elapsed_time(e1) / 10}))
        return
    s.timer = []
    s.advance(steps)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for _, a, b in s.timer]
    rho = s.state.rho
    print(json.dumps({"stage_ms": sum(ms) / len(ms), "pairs": int(s.cnt.sum().item()),
                      "group": s.group, "variant": s.variant,
                      "umax": s.plan.umax if s.plan else None, "rho_sum": float(rho.sum())}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-side", type=int, default=192)
    ap.add_argument("--kernel", default="1.6h")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--one", action="store_true")
    ap.add_argument("--precision", default="fp64")
    args = ap.parse_args()
    if args.one:
        one(args.n_side, args.kernel, args.steps, args.precision)
        return
    variants = [("cell", "global", 1, 4, 0), ("lattice", "global", 1, 4, 0),
                ("lattice", "global", 2, 4, 0), ("lattice", "global", 1, 6, 0),
                ("lattice", "geo", 1, 4, 0), ("lattice", "global", 1, 5, 0)]
    if os.environ.get("TUNE_VARIANTS"):
        variants = [tuple(v.split(":")[:2]) + tuple(int(x) for x in v.split(":")[2:])
                    for v in os.environ["TUNE_VARIANTS"].split(",")]
    for order, kern, g, mb, sw in variants:
        env = dict(os.environ, SPHB_WC_KERNEL=kern, SPHB_WC_GROUP=str(g), SPHB_WC_MINB=str(mb),
                   SPHB_TILE_GROUP=str(g), SPHB_SWIZZLE=str(sw), SPHB_ENGINE_ORDER=order)
        out = subprocess.run([sys.executable, __file__, "--one", "--n-side", str(args.n_side),
                              "--kernel", args.kernel, "--steps", str(args.steps)], env=env,
                             capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        print(json.dumps({"order": order, "kernel": kern, "group": g, "minb": mb, "swizzle": sw,
                          "result": line}), flush=True)


if __name__ == "__main__":
    main()
