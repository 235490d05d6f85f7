"""Sweep launch variants of the TL-SPH passes on C4 (GPU box).

    python scripts/tune_tl.py [--kernel 1.6h] [--variants 0:0,61:81,...]

Each variant (SPHB_TL_VARIANT_A : SPHB_TL_VARIANT_B, minb*10 + unroll, 0 =
default launch) runs in a fresh process; prints one JSON line per variant
with ms/step (CUDA events around graph-replayed steps) and a field checksum.
"""

import argparse
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(kernel, steps):
    sys.path.insert(0, REPO)
    import torch

    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.tlsph import SolidSystem

    cfg = configs.c4_column(kernel=kernel)
    s = SolidSystem(cfg["X0"], cfg["material"], cfg["spec"], cfg["dp"], fixed=cfg["fixed"],
                    cfl=cfg["cfl"])
    s.v = cfg["v0"].copy()
    s.advance(8)                      # captures and replays the step graph
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.advance(steps)
    e1.record()
    torch.cuda.synchronize()
    out = {"ms_per_step": e0.elapsed_time(e1) / steps, "v_sum": float(abs(s.v).sum())}
    # per-launch breakdown: CUDA events around every library call of
    # non-graph steps (launch gaps excluded)
    from paper_2405_05155_b200 import _lib

    real, times = _lib.call, {}

    def timed(name, *a):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        r = real(name, *a)
        ev1.record()
        times.setdefault(name, []).append((ev0, ev1))
        return r

    _lib.call = timed
    s.advance(steps, graph=False)
    torch.cuda.synchronize()
    _lib.call = real
    out["us_per_call"] = {k: round(1e3 * sum(a.elapsed_time(b) for a, b in v) / len(v), 1)
                          for k, v in times.items()}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="1.6h")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--variants", default="0:0,11:11,12:12,61:61,62:62,81:81,82:82")
    ap.add_argument("--one", action="store_true")
    args = ap.parse_args()
    if args.one:
        one(args.kernel, args.steps)
        return
    for v in args.variants.split(","):
        a, b = v.split(":")
        env = dict(os.environ, SPHB_TL_VARIANT_A=a, SPHB_TL_VARIANT_B=b)
        out = subprocess.run([sys.executable, __file__, "--one", "--kernel", args.kernel,
                              "--steps", str(args.steps)], env=env, capture_output=True,
                             text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        print(json.dumps({"kernel": args.kernel, "variant_a": a, "variant_b": b,
                          "result": line}), flush=True)


if __name__ == "__main__":
    main()
