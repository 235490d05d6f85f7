"""Benchmark of the SPH particle-interaction hot path on B200.

Workload (BASELINE.json configs[4], the north star's headline case): the 3D
weakly-compressible Eulerian Taylor-Green vortex, periodic [0, 2pi]^3,
256^3 = 16,777,216 fixed lattice particles, Riemann fluxes with kernel-
gradient correction, FP64.  One "step" = one EulerianSolver midpoint step
(two fused flux stages + device dt).  The truncated kernel (1.6h) is the
headline `value`; the standard 2h leg runs in the same process for the
truncation speed-up.  Inputs (~2.6 GB of particle records) exceed the 126 MB
L2, so no flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--impl reference` times the reference algorithm's CPU implementation (the
C oracle port of the numba loops, all host threads) on a bounded sample of
the same workload (a 64^3 TGV, same per-particle work), and beside it the
unmodified reference package (baseline/_ref, numba) on one core.

One JSON line on rank 0.  Multi-GPU: `--gpus N` launches N ranks itself
(torch.distributed.run on 127.0.0.1, NCCL_DEBUG=INFO) unless it already runs
under torchrun, and refuses to start when fewer than N GPUs are visible.  The
256^3 box is cut into z-slabs of whole cell layers, one per GPU, with a halo
layer exchanged over NCCL after every stage and the dt max all-reduced
(slab.py) — strong scaling of the same 16.8M-particle problem.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time


REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "particle-steps/s and pair-interactions/s at 1.6h vs 2h; % of HBM roofline"
# compulsory FP64 bytes per particle-step for C5 (stage 1: x 24
# + B 48 + rho 8 + mom 24 read, 32 write = 136; stage 2: + U^n 32 = 168)
BYTES_STAGE = {1: 136, 2: 168}
# bytes a stage launch of this implementation must move per particle beyond
# the int32 pass list: own X 32 + B 48 + S 32 + cnt 4 read, S 32 written;
# stage 2 also reads S_n, M_n (64) and writes M (32) — averaged over the two
IMPL_RECORD_BYTES = 32 + 48 + 32 + 4 + 32 + (64 + 32) / 2.0
# the lattice kernel reads neither X, cnt nor a pass list: B 48 + S 32 read,
# S 32 written, stage 2 also S_n, M_n 64 read and M 32 written
LATTICE_RECORD_BYTES = 48 + 32 + 32 + (64 + 32) / 2.0
# uniform-B form (checked: every record's B equals b0 to 1e-12): no B reads
LATTICE_UB_RECORD_BYTES = 32 + 32 + (64 + 32) / 2.0
# FP64 flops per directed pair of the fused stage kernel, from the SASS of
# k_wc_stage<3,1,5> (37 DFMA + 27 DMUL + 13 DADD per pair in the loop body,
# plus the limiter branch ~3; profiles/r01_ncu_c5_256.md v3)
FLOPS_PER_PAIR_EST = 117
# lattice kernel (wc_lattice.cu), FP64 flops per pair from its SASS
# (DFMA = 2): r2 = 4 stencil (919 DFMA + 308 DMUL + 212 DADD) / 32 slots,
# r2 = 6 stencil (2409 DFMA + 741 DMUL + 572 DADD) / 80 slots (round 2,
# folded slot table; profiles/r02_ncu_c5_256.md)
FLOPS_PER_PAIR_LATTICE = {4: 74, 6: 77}
# uniform-B form ((B_i + B_j) gg_k from the slot table): r2 = 4 838 DFMA +
# 214 DMUL + 68 DADD / 32 slots, r2 = 6 2110 DFMA + 502 DMUL + 164 DADD / 80
FLOPS_PER_PAIR_LATTICE_UB = {4: 61, 6: 61}
# isotropic uniform-B form (b0 = beta I), mirror order: r2 = 4 531 DFMA +
# 282 DMUL + 108 DADD / 32 slots, r2 = 6 1287 DFMA + 690 DMUL + 300 DADD / 80
FLOPS_PER_PAIR_LATTICE_IB = {4: 45, 6: 45}


def traffic_per_launch(kernel: str):
    """DRAM bytes per stage launch from a committed ncu capture of this
    kernel (profiles/r*_traffic.json, newest round first), else None."""
    import glob

    for path in sorted(glob.glob(os.path.join(REPO, "profiles", "r*_traffic.json")), reverse=True):
        try:
            with open(path) as f:
                t = json.load(f)
        except (OSError, ValueError):
            continue
        if t.get("kernel") == kernel:
            s = t["stage_launch"]
            return s["dram_bytes_read"] + s["dram_bytes_write"], os.path.basename(path)
    return None, None


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi sampling (-lms 50) of SM clocks / throttle reasons during
    the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.15)            # let the first sample land before timing
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is None:
            return
        time.sleep(0.06)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        self.rows = [[x.strip() for x in line.split(",")] for line in out.splitlines()
                     if line.strip()]

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 2 + k and r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def make_solver(cfg, dist=None, rank=0, world=1, precision="fp64"):
    from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver,
                                                FluidState)

    n = cfg["pos"].shape[0]
    st = FluidState(vol=cfg["vol"], rho=cfg["rho"], mom=cfg["mom"], etot=None, n_interior=n)
    eos = EosParams(WEAKLY_COMPRESSIBLE, rho0=cfg["rho0"], c_art=cfg["c_art"])
    if world > 1:   # z-slabs of the periodic box, NCCL halo exchange (slab.py)
        from paper_2405_05155_b200.slab import slab_eulerian

        return slab_eulerian(cfg["pos"], st, eos, cfg["spec"], rank=rank, world=world, dist=dist,
                             cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
    return EulerianSolver(cfg["pos"], n, st, eos, cfg["spec"], None, correction=True,
                          cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"],
                          precision=precision)


def fp32_leg(torch, cfg, steps, warmup):
    """Optional FP32 mode (north star): its throughput and its error against
    the FP64 engine after the same number of steps from the same state."""
    from paper_2405_05155_b200.approx import l2_error

    s32 = make_solver(cfg, precision="fp32")
    s32.advance(max(warmup, 2), graph=True)        # captures the step graph outside the timing
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s32.advance(steps, graph=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st32 = s32.state
    rho32, mom32 = st32.rho.copy(), st32.mom.copy()
    del s32
    torch.cuda.empty_cache()
    s64 = make_solver(cfg)
    s64.advance(max(warmup, 2) + steps)
    st64 = s64.state
    rho0 = cfg["rho0"]
    err = {"rel_l2_mom": l2_error(mom32, st64.mom),
           "rel_l2_rho_minus_rho0": l2_error(rho32 - rho0, st64.rho - rho0),
           "after_steps": warmup + steps}
    del s64
    torch.cuda.empty_cache()
    n = cfg["pos"].shape[0]
    return {"value": n * steps / (ms * 1e-3), "ms_per_step": ms / steps, "error_vs_fp64": err}


def fp64_peak(torch, lib):
    """Measured DFMA throughput (TFLOP/s) of this GPU: the FP64 roofline."""
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, threads, iters = sms * 8, 256, 20000
    s = torch.cuda.current_stream().cuda_stream
    lib.sphb_fp64_probe(out.data_ptr(), blocks, threads, 2000, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lib.sphb_fp64_probe(out.data_ptr(), blocks, threads, iters, s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return 2.0 * 8 * iters * blocks * threads / (ms * 1e-3) / 1e12


def run_leg(torch, cfg, steps, warmup, dist, world, clocks_index=None):
    """Device-timed K steps of one kernel leg; returns a dict of measurements."""
    rank = dist.get_rank() if dist is not None else 0
    solver = make_solver(cfg, dist, rank, world)
    n = cfg["pos"].shape[0]                          # particles of the whole job
    rows = solver._slab.rows if solver._slab is not None else slice(0, solver.n)
    pairs_t = solver.cnt[rows].sum().to(torch.int64).reshape(1)
    if dist is not None:
        dist.all_reduce(pairs_t)
    pairs = int(pairs_t.item())                      # directed pairs per pass, all ranks
    from paper_2405_05155_b200 import _lib

    before = sum(_lib.CALLS.values())
    solver.advance(1, graph=False)                   # one eager step: count its launches
    launches_per_step = sum(_lib.CALLS.values()) - before
    solver.advance(warmup)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    solver.timer = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(clocks_index) if clocks_index is not None else None
    if sampler:
        sampler.__enter__()
    torch.cuda.synchronize()
    e0.record()
    solver.advance(steps)
    e1.record()
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    st = {1: [], 2: []}
    for stage, a, b in solver.timer:
        st[stage].append(a.elapsed_time(b))
    solver.timer = None
    kernel = {"geo": "k_wc_stage_geo<3>",
              "global": "k_wc_stage<3,%d,%s>" % (solver.group,
                                                 os.environ.get("SPHB_WC_MINB", "5"))}[solver.variant]
    if solver.lattice is not None:
        r4 = solver.lattice.r2 == 4
        kernel = "k_wc_lattice<3,%d,%s>" % (solver.lattice.r2, "3" if r4 else "2,256")
        if solver.lattice.uniform_b:
            form = ("isotropic_b" if solver.lattice_isotropic_b
                    and os.environ.get("SPHB_LAT_IB", "1") != "0" else "uniform_b")
            kernel = "k_wc_lattice<3,%d,%s,%s>" % (solver.lattice.r2, "4" if r4 else "3", form)

    return {"solver": solver, "n": n, "pairs": pairs, "ms": ms, "stage_ms": st, "kernel": kernel,
            "clocks": sampler.summary() if sampler else None,
            "launches_per_step": launches_per_step}


# compulsory FP64 bytes per particle-step of C4 (TL-SPH):
# pass A reads X0 24 + v 24 + a 24 + B0 48 + F 72 + x 24, writes v_half,
# x, F 120; pass B reads X0, F, B0, v_half 168, writes a, v 48
C4_BYTES_STEP = 552


def c4_leg(torch, steps, warmup, peak):
    """Driver-timed sub-record for BASELINE configs[3] (C4, the 3D TL-SPH
    twisting column at dp = 1/68, 1,886,592 particles, FP64): ms per KDK
    step at 1.6h and 2h through SolidSystem.advance (CUDA-graph replay),
    CUDA events, and the HBM fraction on the compulsory bytes."""
    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.tlsph import SolidSystem

    out = {"workload": "c4_column_dp1/68_tl_svk", "unit": "particle-steps/s",
           "bytes_per_particle_step": C4_BYTES_STEP}
    for key in ("1.6h", "2h"):
        cfg = configs.c4_column(kernel=key)
        s = SolidSystem(cfg["X0"], cfg["material"], cfg["spec"], cfg["dp"], fixed=cfg["fixed"],
                        cfl=cfg["cfl"])
        s.v = cfg["v0"]
        s.advance(max(warmup, 8))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = max(steps, 16)
        e0.record()
        s.advance(k)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        n = s.n
        pairs = int(s.cnt.sum().item())
        rec = {"ms_per_step": ms, "value": n / (ms * 1e-3), "particles": n,
               "pair_interactions_per_s": 2 * pairs / (ms * 1e-3), "steps": k,
               "lattice_path": s.lattice is not None}
        if key == "1.6h":
            gbs = C4_BYTES_STEP * n / (ms * 1e-3) / 1e9
            rec["roofline"] = {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                               "frac": gbs / peak}
            ref_state = (s.x - s.X0, s.v, s.F)
            steps_done = s.steps
        out[key.replace(".", "p")] = rec
        del s
        torch.cuda.empty_cache()
        if key == "1.6h":           # optional FP32 mode, its error vs FP64 reported beside
            from paper_2405_05155_b200.approx import l2_error

            s32 = SolidSystem(cfg["X0"], cfg["material"], cfg["spec"], cfg["dp"],
                              fixed=cfg["fixed"], cfl=cfg["cfl"], precision="fp32")
            s32.v = cfg["v0"]
            s32.advance(max(warmup, 8))
            torch.cuda.synchronize()
            e0.record()
            s32.advance(k)
            e1.record()
            torch.cuda.synchronize()
            ms32 = e0.elapsed_time(e1) / k
            assert s32.steps == steps_done
            got = (s32.x - s32.X0, s32.v, s32.F)
            out["fp32_mode_1p6h"] = {
                "ms_per_step": ms32, "value": n / (ms32 * 1e-3),
                "error_vs_fp64": {name: l2_error(a, b) for name, a, b in
                                  zip(("rel_l2_displacement", "rel_l2_v", "rel_l2_F"), got,
                                      ref_state)},
                "after_steps": steps_done,
                "note": "FP32 companions of the gathered v_half / Q records, FP32 pair "
                        "arithmetic flushed to FP64 every 8 slots, FP64 state; reported "
                        "separately, not the headline"}
            del s32
            torch.cuda.empty_cache()
    out["alpha_T1p6h_over_T2h"] = out["1p6h"]["ms_per_step"] / out["2h"]["ms_per_step"]
    return out


def small_configs_leg(torch):
    """Driver-timed sub-records of BASELINE configs[0..2] at their full sizes
    and step counts (CUDA events around the device loop, CUDA-graph replay
    via advance()/run(); set-up and warm-up outside): C1 relaxation (10^4
    particles, 100 LG updates), C2 TGV-2D (200^2, 1000 steps), C3 plate
    (5,200 particles, 2000 steps), each at 1.6h and 2h where the config has
    two kernels.  These are launch/latency bound at 10^4 particles."""
    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver,
                                                FluidState)
    from paper_2405_05155_b200.relaxation import PeriodicRelaxer
    from paper_2405_05155_b200.tlsph import SolidSystem

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    out = {}
    c1 = configs.c1_relax(seed=0)
    rl = PeriodicRelaxer(c1["pos"], c1["relax_spec"], c1["box"], c1["dp"])
    rl.run(5)
    ms = timed(lambda: rl.run(100))
    out["c1_relax"] = {"particles": 10000, "updates": 100, "ms_per_update": ms / 100,
                       "value": 10000 * 100 / (ms * 1e-3)}
    for key in ("1.6h", "2h"):
        cfg = configs.c2_tgv2d(kernel=key)
        n = cfg["pos"].shape[0]
        s = EulerianSolver(cfg["pos"], n, FluidState(cfg["vol"], cfg["rho"], cfg["mom"], None, n),
                           EosParams(WEAKLY_COMPRESSIBLE, rho0=cfg["rho0"], c_art=cfg["c_art"]),
                           cfg["spec"], None, cfl=cfg["cfl"], mu=cfg["mu"],
                           periodic_box=cfg["box"])
        s.advance(16)
        ms = timed(lambda: s.advance(1000))
        out.setdefault("c2_tgv2d", {"particles": n, "steps": 1000})[key.replace(".", "p")] = {
            "ms_per_step": ms / 1000, "value": n * 1000 / (ms * 1e-3)}
        cfg = configs.c3_plate(kernel=key)
        t = SolidSystem(cfg["X0"], cfg["material"], cfg["spec"], cfg["dp"], fixed=cfg["fixed"],
                        cfl=cfg["cfl"])
        t.v = cfg["v0"]
        t.advance(16)
        ms = timed(lambda: t.advance(2000))
        out.setdefault("c3_plate", {"particles": t.n, "steps": 2000})[key.replace(".", "p")] = {
            "ms_per_step": ms / 2000, "value": t.n * 2000 / (ms * 1e-3)}
    for name in ("c2_tgv2d", "c3_plate"):
        out[name]["alpha_T1p6h_over_T2h"] = (out[name]["1p6h"]["ms_per_step"]
                                             / out[name]["2h"]["ms_per_step"])
    return out


def e2e_leg(torch, solver, steps, warmup):
    """Through the public API with host buffers: every step uploads a state
    from pinned host memory (EulerianSolver.load_state), advances one step and
    reads the new state back into pinned host memory (read_state) — both
    copies of every step inside the timed region.  Input and output host
    buffers are distinct (a stream of independent one-step problems), so the
    state transfers run on their own copy streams: the next step's input is
    prefetched (prefetch_state) while the step computes and one step's
    device-to-host copy overlaps the next step's host-to-device copy
    (read_state(wait=False)).  The timed region holds K host-to-device and K
    device-to-host copies: the end event waits for the last read and for the
    prefetch the last step issued (step 1's input was staged before e0)."""
    n, d = solver.n, solver.dim
    rho_in = torch.empty(n, dtype=torch.float64).pin_memory()
    mom_in = torch.empty((n, d), dtype=torch.float64).pin_memory()
    rho_out = torch.empty(n, dtype=torch.float64).pin_memory()
    mom_out = torch.empty((n, d), dtype=torch.float64).pin_memory()
    solver.read_state(rho_in, mom_in)
    torch.cuda.synchronize()
    last = []

    def one():
        solver.load_state(rho_in, mom_in)
        solver.prefetch_state(rho_in, mom_in)    # next step's input, during this step
        solver.step()                 # the reference API call (eulerian.py:562)
        last[:] = [solver.read_state(rho_out, mom_out, wait=False)]

    solver.prefetch_state(rho_in, mom_in)
    for _ in range(warmup):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        one()
    # the region holds K host-to-device copies: step 1's input was staged
    # before e0, so the prefetch issued by step K is waited for as well
    torch.cuda.current_stream().wait_event(last[0])
    torch.cuda.current_stream().wait_event(solver._io["prefetched"][2])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    nbytes = rho_in.numel() * 8 + mom_in.numel() * 8
    return ms / steps, nbytes


def cpu_reference(kind_n_side=64, steps=3, kernel="1.6h"):
    """The reference algorithm on the host cores: oracle port (C loops of the
    numba kernels + numpy glue), all OpenMP threads, TGV-3D at n_side^3."""
    from oracle import oracle as O
    from paper_2405_05155_b200 import configs

    cfg = configs.c5_tgv3d(kernel=kernel, n_side=kind_n_side)
    s = O.EulerianWC(cfg["pos"], cfg["vol"], cfg["rho"], cfg["mom"], cfg["spec"], cfg["c_art"],
                     cfg["rho0"], cfg["mu"], cfg["cfl"], cfg["box"])
    s.rhs()                                          # warm-up (bench.py:94-105 protocol)
    t0 = time.perf_counter()
    for _ in range(steps):
        s.step()
    dt = time.perf_counter() - t0
    n = cfg["pos"].shape[0]
    return {"value": n * steps / dt, "unit": "particle-steps/s", "cores": O.threads(),
            "kind": "port", "pairs_per_s": int(s.nl.starts[-1]) * 2 * steps / dt,
            "sample": f"TGV-3D {kind_n_side}^3 ({n} particles, {kernel}), {steps} steps after one "
                      "warm-up rhs; same per-particle work as 256^3"}


def free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return int(sk.getsockname()[1])


def visible_gpus() -> int:
    try:
        import torch

        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:           # noqa: BLE001 - a broken runtime counts as no GPU
        return 0


def launch(args) -> int:
    """`--gpus N` (N > 1) run without torchrun: start N ranks of this script,
    one per GPU, under torch.distributed.run on 127.0.0.1 (the driver's own
    launch form).  Refuses to run when fewer than N GPUs are visible instead
    of silently timing fewer."""
    if not args.launch_check:
        have = visible_gpus()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}",
                  file=sys.stderr)
            return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")        # communicator lines in the log
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def launch_check(world, rank):
    """Rank body of `--launch-check`: gloo on CPU, one all_reduce, rank 0
    prints what the launcher started (tests/test_bench_launch.py)."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    t = torch.tensor([1 << rank], dtype=torch.int64)
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": dist.get_world_size(),
                          "ranks_mask": int(t.item()),
                          "master_addr": os.environ.get("MASTER_ADDR"),
                          "nccl_debug": os.environ.get("NCCL_DEBUG")}))
    dist.destroy_process_group()


def numba_reference(n_side=64, steps=2, kernel="1.6h"):
    """The reference package itself (sph_trunc from baseline/_ref, its numba
    kernels) on ONE host core, as BASELINE.md §3 planned: build outside the
    timer, one warm-up rhs (its bench.py:94-105), then `steps` EulerianSolver
    steps.  None when baseline/_ref or numba is missing."""
    ref_dir = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "sph_trunc")):
        return None
    code = f"""
import os, sys, time, json
os.sched_setaffinity(0, {{min(os.sched_getaffinity(0))}})
sys.path.insert(0, {ref_dir!r}); sys.path.insert(1, {REPO!r})
from sph_trunc import eulerian
from paper_2405_05155_b200 import configs
cfg = configs.c5_tgv3d(kernel={kernel!r}, n_side={n_side})
n = cfg["pos"].shape[0]
st = eulerian.FluidState(vol=cfg["vol"].copy(), rho=cfg["rho"].copy(), mom=cfg["mom"].copy(),
                         etot=None, n_interior=n)
eos = eulerian.EosParams(eulerian.WEAKLY_COMPRESSIBLE, rho0=cfg["rho0"], c_art=cfg["c_art"])
s = eulerian.EulerianSolver(cfg["pos"], n, st, eos, cfg["spec"], None, correction=True,
                            cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
s.rhs()
t0 = time.perf_counter()
for _ in range({steps}):
    s.step()
dt = time.perf_counter() - t0
print(json.dumps({{"value": n * {steps} / dt, "pairs": int(s.nlist.starts[-1])}}))
"""
    env = dict(os.environ, NUMBA_NUM_THREADS="1", OMP_NUM_THREADS="1",
               OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                             text=True, timeout=900)
        r = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as exc:    # noqa: BLE001 - reported, not fatal
        return {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    return {"value": r["value"], "unit": "particle-steps/s", "cores": 1, "kind": "reference",
            "pairs_per_s": r["pairs"] * 2 * steps / (n_side**3 * steps / r["value"]),
            "sample": f"sph_trunc (numba, the unmodified reference from baseline/_ref) on one "
                      f"pinned core, TGV-3D {n_side}^3 {kernel}, {steps} steps after one warm-up "
                      "rhs"}


def reference_arm(args, config):
    """`--impl reference`: the reference algorithm on this box's host cores.
    The line's value is the oracle port (the numba loops restated in C, all
    OpenMP threads: the stronger CPU baseline); the unmodified single-core
    reference package is reported beside it.  Both time a bounded 64^3
    sample of the 256^3 workload (same per-particle work: the lattice, h/dp
    and pair count per particle do not depend on the box size)."""
    warm = max(0, args.warmup)
    steps = max(1, args.steps)
    ref = cpu_reference(steps=steps)
    ms = 1e3 * (64**3) / ref["value"]
    cfg = dict(config, sample="TGV-3D 64^3 (262,144 particles) of the 256^3 workload",
               particles=64**3, particles_per_gpu=64**3, parallelism="host CPU")
    line = {"metric": METRIC, "value": ref["value"], "unit": "particle-steps/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": steps, "warmup": warm,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": ref["value"], "unit": "particle-steps/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "pair_interactions_per_s": ref["pairs_per_s"]}
    if not args.no_numba:
        nb = numba_reference()
        if nb is not None:
            line["reference_package_1core"] = nb
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-side", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-2h", action="store_true")
    ap.add_argument("--no-fp32", action="store_true")
    ap.add_argument("--no-c4", action="store_true",
                    help="skip the C1-C4 sub-records (small configs and the TL-SPH column)")
    ap.add_argument("--no-numba", action="store_true",
                    help="reference arm: skip the single-core sph_trunc (numba) figure")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and (args.impl == "ours"
                                                            or args.launch_check):
        sys.exit(launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.launch_check:
        launch_check(world, rank)
        return
    if args.impl == "ours" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    config = {"workload": f"c5_tgv3d_{args.n_side}^3_wc_euler_riemann_corrected",
              "particles": args.n_side**3,
              "particles_per_gpu": args.n_side**3 // max(1, world),
              "kernel": "wendland C2 truncated 1.6h",
              "steps_definition": "one midpoint step = 2 fused flux stages",
              "l2": "inputs > L2 (126 MB); no flush",
              "parallelism": "single GPU" if world == 1 else f"z-slabs x{world}, NCCL halo"}

    if args.impl == "reference":
        if rank != 0:
            return
        reference_arm(args, config)
        return

    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    from paper_2405_05155_b200 import _lib, configs

    lib = _lib.lib()
    pk, pk_kind = peaks()
    fp64_tf = fp64_peak(torch, lib)

    leg = {}
    cfg = configs.c5_tgv3d(kernel="1.6h", n_side=args.n_side)
    leg["1.6h"] = run_leg(torch, cfg, args.steps, max(3, args.warmup), dist, world,
                          clocks_index=local)
    e2e_ms, io_bytes = e2e_leg(torch, leg["1.6h"]["solver"], max(4, args.steps // 2), 2)
    sv = leg["1.6h"]["solver"]          # this GPU's rows (owned + halo)
    design_bytes = sv.n * (IMPL_RECORD_BYTES + 4.0 * sv.width)
    flops_pair = FLOPS_PER_PAIR_EST
    # which specialisations of the stage this run proved and used (each is
    # checked on the device before use)
    config["stage_path"] = "general pass-list kernel"
    if sv.lattice is not None:
        config["stage_path"] = ("lattice: computed neighbour indices, per-slot geometry table "
                                "(pair sets and displacements checked per row to 1e-12 dp)")
        if sv.lattice.uniform_b:
            config["stage_path"] += ("; uniform B (every B_i = b0 to 1e-12, checked), "
                                     + ("b0 = beta I: isotropic form, mirror order"
                                        if sv.lattice_isotropic_b else "per-slot (B_i+B_j) gg"))
        design_bytes = sv.n * LATTICE_RECORD_BYTES
        flops_pair = FLOPS_PER_PAIR_LATTICE[sv.lattice.r2]
        if sv.lattice.uniform_b:
            design_bytes = sv.n * LATTICE_UB_RECORD_BYTES
            flops_pair = FLOPS_PER_PAIR_LATTICE_UB[sv.lattice.r2]
            if sv.lattice_isotropic_b and os.environ.get("SPHB_LAT_IB", "1") != "0":
                flops_pair = FLOPS_PER_PAIR_LATTICE_IB[sv.lattice.r2]
    del leg["1.6h"]["solver"], sv
    torch.cuda.empty_cache()
    if not args.no_2h:
        cfg2 = configs.c5_tgv3d(kernel="2h", n_side=args.n_side)
        leg["2h"] = run_leg(torch, cfg2, args.steps, max(3, args.warmup), dist, world)
        del leg["2h"]["solver"]
        torch.cuda.empty_cache()
    small = None
    if world == 1 and not args.no_c4:
        small = small_configs_leg(torch)
    c4 = None
    if world == 1 and not args.no_c4:
        c4 = c4_leg(torch, args.steps, args.warmup, float(peaks()[0]["hbm_gbs"]))
    f32 = None
    if world == 1 and not args.no_fp32:
        f32 = fp32_leg(torch, cfg, args.steps, max(3, args.warmup))

    L = leg["1.6h"]
    n, K = L["n"], args.steps
    ms_step = L["ms"] / K
    value = n * K / (L["ms"] * 1e-3)                 # whole job (n = all ranks' particles)
    stage_all = L["stage_ms"][1] + L["stage_ms"][2]
    avg_stage_ms = sum(stage_all) / len(stage_all)
    alg_bytes = n / world * (BYTES_STAGE[1] + BYTES_STAGE[2]) / 2.0  # per launch, per GPU
    achieved = alg_bytes / (avg_stage_ms * 1e-3) / 1e9
    hbm_peak = float(pk["hbm_gbs"])
    traffic = traffic_per_launch(L["kernel"]) if world == 1 else (None, None)
    fp64_ach = L["pairs"] / world * flops_pair / (avg_stage_ms * 1e-3) / 1e12

    line = {
        "metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": world,
        "steps": K, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic TGV-3D fields on the 256^3 lattice)", "config": config,
        "pair_interactions_per_s": L["pairs"] * 2 * K / (L["ms"] * 1e-3),
        "pairs_per_pass": L["pairs"],
        "gpu_launches": L["launches_per_step"] * K,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak,
                     "traffic": traffic[0], "traffic_source": traffic[1],
                     "kernel": L["kernel"], "peak_kind": pk_kind,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     # what the traffic should be for this design: own records
                     # once + the int32 pass list (SURVEY's compulsory bytes
                     # leave the list out), i.e. no neighbour re-reads
                     "design_bytes_per_launch": design_bytes,
                     "avg_launch_ms": avg_stage_ms,
                     "stage_ms": {"1": statistics.mean(L["stage_ms"][1]),
                                  "2": statistics.mean(L["stage_ms"][2])},
                     "fp64": {"achieved_tflops_est": fp64_ach, "peak_tflops_measured": fp64_tf,
                              "frac": fp64_ach / fp64_tf,
                              "flops_per_pair_est": flops_pair}},
        "clocks": L["clocks"],
        "e2e": {"value": n / (e2e_ms * 1e-3), "unit": "particle-steps/s",
                "h2d_bytes_per_step": io_bytes, "d2h_bytes_per_step": io_bytes,
                "ms_per_step": e2e_ms,
                "path": ("EulerianSolver.load_state(pinned) -> prefetch_state(next) -> "
                         "step() -> read_state(pinned, wait=False); copy streams, "
                         "transfers overlap the step and each other")},
    }
    if world > 1:
        # per-GPU view of the slab run: stage kernels vs the step; the rest
        # is the exposed halo exchange + dt all-reduce + launch gaps
        stage_step = statistics.mean(L["stage_ms"][1]) + statistics.mean(L["stage_ms"][2])
        line["per_gpu"] = {"stage_ms_per_step": stage_step, "ms_per_step": ms_step,
                           "exposed_comm_ms_per_step": max(0.0, ms_step - stage_step),
                           "exposed_comm_share": max(0.0, ms_step - stage_step) / ms_step,
                           "particles_owned": n // world}
    if "2h" in leg:
        S = leg["2h"]
        line["standard_2h"] = {
            "value": S["n"] * K / (S["ms"] * 1e-3), "ms_per_step": S["ms"] / K,
            "pair_interactions_per_s": S["pairs"] * 2 * K / (S["ms"] * 1e-3),
            "pairs_per_pass": S["pairs"], "kernel": S["kernel"]}
        line["alpha_T1p6h_over_T2h"] = L["ms"] / S["ms"]
    if c4 is not None:
        line["c4_column"] = c4
    if small is not None:
        line["small_configs"] = small
    if f32 is not None:
        line["fp32_mode"] = dict(f32, unit="particle-steps/s", kernel="k_wc_lattice_f32<3,4>",
                                 note="FP32 pair math, FP64 accumulation/state; reported "
                                      "separately, not the headline")
    if rank == 0 and not args.no_cpu_baseline:
        cb = cpu_reference()
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
