"""Slab-decomposed WC solver on ONE GPU: ranks as host threads.

The NCCL path cannot be exercised with one GPU (and ranks whose kernels wait
on one another must not share a GPU), so each simulated rank runs in its own
host thread with its own CUDA stream and solver, and a thread-rendezvous
stand-in for torch.distributed performs the halo copies and the dt all-reduce
between them.  No kernel ever waits on another rank: the host threads meet
at a barrier after synchronising their streams.  The owned rows gathered from
all ranks must equal the single-GPU solver's rows.
"""

import threading
from collections import defaultdict

import numpy as np
import pytest
import torch

from paper_2405_05155_b200 import configs
from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver,
                                            FluidState)
from paper_2405_05155_b200.slab import slab_eulerian

pytestmark = pytest.mark.gpu


class _Op:
    def __init__(self, fn, tensor, peer, group=None):
        self.fn, self.tensor, self.peer = fn, tensor, peer


class ThreadDist:
    """Per-rank view of a shared rendezvous that mimics the torch.distributed
    calls slab.py and eulerian.py make (P2POp, batch_isend_irecv,
    all_reduce MAX)."""

    class ReduceOp:
        MAX = "max"
        SUM = "sum"

    P2POp = _Op

    def __init__(self, shared, rank):
        self.shared, self.rank = shared, rank

    def isend(self, *a):  # sentinels
        raise AssertionError

    def irecv(self, *a):
        raise AssertionError

    def batch_isend_irecv(self, ops):
        sh = self.shared
        torch.cuda.current_stream().synchronize()
        count = defaultdict(int)
        for op in ops:
            if op.fn == self.isend:
                k = count[("s", op.peer)]
                count[("s", op.peer)] += 1
                with sh.lock:
                    sh.box[(self.rank, op.peer, k)] = op.tensor
        sh.barrier.wait()
        count.clear()
        for op in ops:
            if op.fn == self.irecv:
                k = count[("r", op.peer)]
                count[("r", op.peer)] += 1
                src = sh.box[(op.peer, self.rank, k)]
                assert src.shape == op.tensor.shape
                op.tensor.copy_(src)
        torch.cuda.current_stream().synchronize()
        sh.barrier.wait()
        if self.rank == 0:
            sh.box.clear()
        sh.barrier.wait()
        return []

    def get_rank(self):
        return self.rank

    def get_world_size(self):
        return self.shared.world

    def share_device_buffers(self, ptrs, halo):
        """Fused halo push: every rank's buffer pointers (same device)."""
        sh = self.shared
        with sh.lock:
            sh.ptrs[self.rank] = (list(ptrs), tuple(halo))
        sh.barrier.wait()
        table = dict(sh.ptrs)
        sh.barrier.wait()
        return table

    def barrier(self):
        torch.cuda.current_stream().synchronize()
        self.shared.barrier.wait()

    def all_reduce(self, t, op="sum"):
        sh = self.shared
        torch.cuda.current_stream().synchronize()
        with sh.lock:
            sh.red[self.rank] = t.clone()
        sh.barrier.wait()
        vals = torch.stack([sh.red[r] for r in range(sh.world)])
        t.copy_(vals.max(dim=0).values if op == "max" else vals.sum(dim=0))
        torch.cuda.current_stream().synchronize()
        sh.barrier.wait()


class Shared:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.lock = threading.Lock()
        self.box = {}
        self.red = {}
        self.ptrs = {}


def _state(cfg):
    n = cfg["pos"].shape[0]
    return FluidState(cfg["vol"].copy(), cfg["rho"].copy(), cfg["mom"].copy(), None, n)


@pytest.mark.parametrize("mode", ["exchange", "overlap", "push"])
@pytest.mark.parametrize("world,kernel", [(2, "1.6h"), (3, "2h"), (4, "1.6h")])
def test_slab_solver_matches_single_gpu(monkeypatch, world, kernel, mode):
    """Owned rows of every rank equal the single-GPU solver's: with the P2P
    exchange after each stage, with boundary-first stages whose exchange runs
    on a side stream under the interior rows (the default), and with `push`
    (the stage kernels store the boundary layers straight into the neighbour
    ranks' halo rows, SPHB_HALO_PUSH=1)."""
    push = mode == "push"
    monkeypatch.setenv("SPHB_HALO_PUSH", "1" if push else "0")
    monkeypatch.setenv("SPHB_SLAB_OVERLAP", "1" if mode == "overlap" else "0")
    cfg = configs.c5_tgv3d(kernel=kernel, n_side=24)
    eos = EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=cfg["c_art"])
    steps = 5
    ref = EulerianSolver(cfg["pos"], cfg["pos"].shape[0], _state(cfg), eos, cfg["spec"], None,
                         cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
    ref.advance(steps)
    want_rho, want_mom = ref.state.rho, ref.state.mom

    shared = Shared(world)
    results, errors, lattice = {}, [], {}

    def run(rank):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                d = ThreadDist(shared, rank)
                s = slab_eulerian(cfg["pos"], _state(cfg), eos, cfg["spec"], rank=rank,
                                  world=world, dist=d, cfl=cfg["cfl"], mu=cfg["mu"],
                                  periodic_box=cfg["box"])
                assert (s._push is not None) == push
                assert (s._overlap is not None) == (mode == "overlap")
                lattice[rank] = s.lattice is not None      # checked per rank (owned rows)
                s.advance(steps)
                results[rank] = s.owned()
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)
            shared.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    # the TGV slabs are lattices: every rank runs the WC lattice kernel
    assert ref.lattice is not None and all(lattice.values()), lattice
    got_rho = np.full_like(want_rho, np.nan)
    got_mom = np.full_like(want_mom, np.nan)
    for ids, rho, mom in results.values():
        got_rho[ids] = rho
        got_mom[ids] = mom
    assert not np.isnan(got_rho).any()
    # identical rows and summation order; only FMA scheduling may differ
    np.testing.assert_allclose(got_rho, want_rho, rtol=1e-14, atol=0)
    np.testing.assert_allclose(got_mom, want_mom, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("push", [False, True])
@pytest.mark.parametrize("world,kernel", [(2, "1.6h"), (3, "2h")])
def test_slab_solid_matches_single_gpu(monkeypatch, world, kernel, push):
    """Owned rows equal the single-GPU system's; with `push` the pass A / B
    epilogues write the Q, a and v halos into the neighbours' rows."""
    from paper_2405_05155_b200.slab import slab_solid
    from paper_2405_05155_b200.tlsph import SolidSystem

    cfg = configs.c4_column(kernel=kernel, n_width=6)
    steps = 20
    monkeypatch.setenv("SPHB_HALO_PUSH", "1" if push else "0")
    ref = SolidSystem(cfg["X0"], cfg["material"], cfg["spec"], cfg["dp"], fixed=cfg["fixed"],
                      cfl=cfg["cfl"])
    ref.v = cfg["v0"]
    ref.advance(steps)
    want = (ref.x, ref.v, ref.F)

    shared = Shared(world)
    results, errors = {}, []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                d = ThreadDist(shared, rank)
                s = slab_solid(cfg["X0"], cfg["material"], cfg["spec"], cfg["dp"], rank=rank,
                               world=world, dist=d, fixed=cfg["fixed"], cfl=cfg["cfl"])
                assert s._slab.axis == 1          # the column's long axis
                assert (s._push is not None) == push
                s.v = cfg["v0"][s.local_ids]
                s.advance(steps)
                results[rank] = s.owned()
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover
            errors.append(e)
            shared.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    got = [np.full_like(w, np.nan) for w in want]
    for ids, x, v, F in results.values():
        for g, val in zip(got, (x, v, F)):
            g[ids] = val
    for g, w in zip(got, want):
        assert not np.isnan(g).any()
        np.testing.assert_allclose(g, w, rtol=1e-12, atol=1e-14 * np.abs(w).max())


def test_bench_multi_rank_leg_with_thread_ranks():
    """bench.py's multi-GPU leg (slab solver, barrier, max-over-ranks time,
    all-reduced pair count) driven by two thread ranks on one GPU."""
    import bench

    cfg = configs.c5_tgv3d(n_side=24)
    world = 2
    shared = Shared(world)
    out, errors = {}, []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                d = ThreadDist(shared, rank)
                out[rank] = bench.run_leg(torch, cfg, 3, 3, d, world)
        except Exception as e:  # pragma: no cover
            errors.append(e)
            shared.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    assert out[0]["pairs"] == out[1]["pairs"] == 24**3 * 32
    assert out[0]["ms"] == out[1]["ms"] > 0.0
