"""Throughput of all five BASELINE configs at 1.6h and 2h (GPU) beside the
CPU oracle port (all host threads).  One JSON line per (config, kernel).

    python scripts/bench_configs.py [--configs c1,c2,c3,c4,c5] [--cpu]

Units: particle-steps/s = N steps / s; pair-interactions/s =
directed pairs x passes per step x steps / s (WC: 2 stages, TL: dF + acc,
relaxation: 1).  GPU times are CUDA-event times of the step loop after
warm-up, CUDA-graph replay (the engines' advance()/run()).
"""

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def timed(torch, fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def wc(torch, cfg, steps):
    from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver,
                                                FluidState)

    n = cfg["pos"].shape[0]
    s = EulerianSolver(cfg["pos"], n, FluidState(cfg["vol"], cfg["rho"], cfg["mom"], None, n),
                       EosParams(WEAKLY_COMPRESSIBLE, rho0=cfg["rho0"], c_art=cfg["c_art"]),
                       cfg["spec"], None, cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
    s.advance(10)
    sec = timed(torch, lambda: s.advance(steps))
    return n, int(s.cnt.sum().item()), 2, sec


def tl(torch, cfg, steps):
    from paper_2405_05155_b200.tlsph import SolidSystem

    s = SolidSystem(cfg["X0"], cfg["material"], cfg["spec"], cfg["dp"], fixed=cfg["fixed"],
                    cfl=cfg["cfl"])
    s.v = cfg["v0"]
    s.advance(10)
    sec = timed(torch, lambda: s.advance(steps))
    return cfg["X0"].shape[0], int(s.cnt.sum().item()), 2, sec


def cpu_wc(cfg, steps):
    from oracle import oracle as O

    s = O.EulerianWC(cfg["pos"], cfg["vol"], cfg["rho"], cfg["mom"], cfg["spec"], cfg["c_art"],
                     cfg["rho0"], cfg["mu"], cfg["cfl"], cfg["box"])
    s.rhs()
    t0 = time.perf_counter()
    for _ in range(steps):
        s.step()
    return time.perf_counter() - t0, int(s.nl.starts[-1])


def cpu_tl(cfg, steps):
    from oracle import oracle as O

    m = cfg["material"]
    s = O.SolidTL(cfg["X0"], m.rho0, m.E, m.nu, cfg["spec"], cfg["dp"], cfg["fixed"], True,
                  cfg["cfl"])
    s.v = cfg["v0"].copy()
    s.accelerations()
    t0 = time.perf_counter()
    for _ in range(steps):
        s.step()
    return time.perf_counter() - t0, int(s.nl.starts[-1])


def emit(**kw):
    print(json.dumps(kw), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--cpu", action="store_true", help="also time the CPU oracle port")
    args = ap.parse_args()
    import torch

    from oracle import oracle as O
    from paper_2405_05155_b200 import configs, neighbors
    from paper_2405_05155_b200.approx import sph_unity_sum_device
    from paper_2405_05155_b200.relaxation import PeriodicRelaxer

    todo = args.configs.split(",")
    threads = O.threads()
    if "c1" in todo:
        c1 = configs.c1_relax(seed=0)
        rl = PeriodicRelaxer(c1["pos"], c1["relax_spec"], c1["box"], c1["dp"])
        rl.run(5)
        sec = timed(torch, lambda: rl.run(100))
        nl = neighbors.build_neighbors(c1["pos"], c1["relax_spec"].kappa * c1["h"], c1["box"])
        emit(config="c1_relax", kernel="LG kappa=2", n=10000, steps=100, seconds=sec,
             particle_steps_per_s=10000 * 100 / sec, pair_int_per_s=nl.m * 100 / sec)
        pos_final = rl.positions()
        vols = np.full(10000, c1["vol"])
        for key, spec in configs.density_specs(c1["h"]).items():
            def dens():
                nl2 = neighbors.build_neighbors(pos_final, spec.kappa * spec.h, c1["box"])
                sph_unity_sum_device(nl2, vols, spec)
            dens()
            sec = timed(torch, dens)
            emit(config="c1_density", kernel=key, n=10000, seconds_build_plus_sum=sec)
        if args.cpu:
            t0 = time.perf_counter()
            O.relax_steps(c1["pos"], c1["relax_spec"], c1["box"], c1["dp"], 100)
            sec = time.perf_counter() - t0
            emit(config="c1_relax", impl="cpu-oracle", threads=threads, seconds=sec,
                 particle_steps_per_s=10000 * 101 / sec)
    for key in ("1.6h", "2h"):
        if "c2" in todo:
            cfg = configs.c2_tgv2d(kernel=key)
            n, m, passes, sec = wc(torch, cfg, 1000)
            emit(config="c2_tgv2d", kernel=key, n=n, steps=1000, seconds=sec,
                 particle_steps_per_s=n * 1000 / sec, pair_int_per_s=m * passes * 1000 / sec)
            if args.cpu:
                sec, m = cpu_wc(cfg, 100)
                emit(config="c2_tgv2d", kernel=key, impl="cpu-oracle", threads=threads, steps=100,
                     particle_steps_per_s=n * 100 / sec, pair_int_per_s=m * 2 * 100 / sec)
        if "c3" in todo:
            cfg = configs.c3_plate(kernel=key)
            n, m, passes, sec = tl(torch, cfg, 2000)
            emit(config="c3_plate", kernel=key, n=n, steps=2000, seconds=sec,
                 particle_steps_per_s=n * 2000 / sec, pair_int_per_s=m * passes * 2000 / sec)
            if args.cpu:
                sec, m = cpu_tl(cfg, 200)
                emit(config="c3_plate", kernel=key, impl="cpu-oracle", threads=threads,
                     steps=200, particle_steps_per_s=n * 200 / sec,
                     pair_int_per_s=m * 2 * 200 / sec)
        if "c4" in todo:
            cfg = configs.c4_column(kernel=key)
            n, m, passes, sec = tl(torch, cfg, 100)
            emit(config="c4_column", kernel=key, n=n, steps=100, seconds=sec,
                 particle_steps_per_s=n * 100 / sec, pair_int_per_s=m * passes * 100 / sec,
                 hbm_gbs_at_552B=552 * n * 100 / sec / 1e9)
            if args.cpu:
                small = configs.c4_column(kernel=key, n_width=20)
                sec, m = cpu_tl(small, 5)
                ns = small["X0"].shape[0]
                emit(config="c4_column", kernel=key, impl="cpu-oracle", threads=threads,
                     sample="dp=1/20 (48k particles), 5 steps", particle_steps_per_s=ns * 5 / sec,
                     pair_int_per_s=m * 2 * 5 / sec)
        if "c5" in todo:
            cfg = configs.c5_tgv3d(kernel=key)
            n, m, passes, sec = wc(torch, cfg, 20)
            emit(config="c5_tgv3d", kernel=key, n=n, steps=20, seconds=sec,
                 particle_steps_per_s=n * 20 / sec, pair_int_per_s=m * passes * 20 / sec,
                 hbm_gbs_at_304B=304 * n * 20 / sec / 1e9)
            del cfg
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
