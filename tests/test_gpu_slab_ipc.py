"""Fused halo push (WC stage and TL passes) across PROCESSES on one GPU: the CUDA-IPC mapping of
SlabPlan.share_buffers (the path torchrun ranks take) with two processes
sharing cuda:0.  The collectives run over gloo on host copies (an adapter
below), so no kernel ever waits on another process: each step's ordering is
a host-side collective after a stream synchronisation.  The owned rows of
both ranks must equal the single-process solver's.  On a box with two or
more GPUs the `two-gpus` variants put the ranks on cuda:0 and cuda:1, so the
pushes are real peer writes over NVLink (skipped on one GPU)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


class HostCollectives:
    """torch.distributed (gloo) with CUDA tensors staged through host copies."""

    class ReduceOp:
        MAX = dist.ReduceOp.MAX
        SUM = dist.ReduceOp.SUM

    P2POp = dist.P2POp
    isend = staticmethod(dist.isend)
    irecv = staticmethod(dist.irecv)

    def batch_isend_irecv(self, ops):
        torch.cuda.current_stream().synchronize()
        host, back = [], []
        for op in ops:
            h = op.tensor.detach().cpu().contiguous()
            host.append(dist.P2POp(op.op, h, op.peer))
            if op.op == dist.irecv:
                back.append((op.tensor, h))
        for req in dist.batch_isend_irecv(host):
            req.wait()
        for dst, h in back:
            dst.copy_(h)
        return []

    def all_reduce(self, t, op=dist.ReduceOp.SUM):
        torch.cuda.current_stream().synchronize()
        h = t.detach().cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)

    def all_gather_object(self, out, obj):
        dist.all_gather_object(out, obj)

    def barrier(self):
        torch.cuda.current_stream().synchronize()
        dist.barrier()

    def get_rank(self):
        return dist.get_rank()

    def get_world_size(self):
        return dist.get_world_size()


def _rank(rank, world, port, out_dir, distinct=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SPHB_HALO_PUSH="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(rank if distinct else 0)
        from paper_2405_05155_b200 import configs
        from paper_2405_05155_b200.eulerian import WEAKLY_COMPRESSIBLE, EosParams, FluidState
        from paper_2405_05155_b200.slab import slab_eulerian

        cfg = configs.c5_tgv3d(kernel="1.6h", n_side=24)
        n = cfg["pos"].shape[0]
        st = FluidState(cfg["vol"].copy(), cfg["rho"].copy(), cfg["mom"].copy(), None, n)
        s = slab_eulerian(cfg["pos"], st, EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0),
                          cfg["spec"], rank=rank, world=world, dist=HostCollectives(),
                          cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
        assert s._push is not None and s._slab._ipc_keep
        s.advance(5)
        ids, rho, mom = s.owned()
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), ids=ids, rho=rho, mom=mom)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _solid_rank(rank, world, port, out_dir, distinct=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SPHB_HALO_PUSH="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(rank if distinct else 0)
        from paper_2405_05155_b200 import configs
        from paper_2405_05155_b200.slab import slab_solid

        cfg = configs.c4_column(kernel="1.6h", n_width=6)
        s = slab_solid(cfg["X0"], cfg["material"], cfg["spec"], cfg["dp"], rank=rank,
                       world=world, dist=HostCollectives(), fixed=cfg["fixed"], cfl=cfg["cfl"])
        assert s._push is not None and s._slab._ipc_keep
        s.v = cfg["v0"][s.local_ids]
        s.advance(10)
        ids, x, v, F = s.owned()
        np.savez(os.path.join(out_dir, f"s{rank}.npz"), ids=ids, x=x, v=v, F=F)
        dist.barrier()
    finally:
        dist.destroy_process_group()


_DEVICES = [pytest.param(False, id="one-gpu"),
            pytest.param(True, id="two-gpus", marks=pytest.mark.skipif(
                torch.cuda.device_count() < 2, reason="needs two GPUs (peer writes over NVLink)"))]


@pytest.mark.parametrize("distinct", _DEVICES)
def test_halo_push_over_cuda_ipc(tmp_path, distinct):
    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver,
                                                FluidState)

    cfg = configs.c5_tgv3d(kernel="1.6h", n_side=24)
    n = cfg["pos"].shape[0]
    ref = EulerianSolver(cfg["pos"], n, FluidState(cfg["vol"].copy(), cfg["rho"].copy(),
                                                   cfg["mom"].copy(), None, n),
                         EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0), cfg["spec"], None,
                         cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
    ref.advance(5)
    want = ref.state
    world = 2
    mp.start_processes(_rank, args=(world, 29511 + int(distinct), str(tmp_path), distinct),
                       nprocs=world, join=True,
                       start_method="spawn")
    got_rho = np.full(n, np.nan)
    got_mom = np.full((n, 3), np.nan)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        got_rho[z["ids"]] = z["rho"]
        got_mom[z["ids"]] = z["mom"]
    assert not np.isnan(got_rho).any()
    np.testing.assert_allclose(got_rho, want.rho, rtol=1e-14, atol=0)
    np.testing.assert_allclose(got_mom, want.mom, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("distinct", _DEVICES)
def test_solid_halo_push_over_cuda_ipc(tmp_path, distinct):
    """TL-SPH: pass A pushes Q, pass B pushes a and v across processes."""
    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.tlsph import SolidSystem

    cfg = configs.c4_column(kernel="1.6h", n_width=6)
    ref = SolidSystem(cfg["X0"], cfg["material"], cfg["spec"], cfg["dp"], fixed=cfg["fixed"],
                      cfl=cfg["cfl"])
    ref.v = cfg["v0"]
    ref.advance(10)
    want = (ref.x, ref.v, ref.F)
    world = 2
    mp.start_processes(_solid_rank, args=(world, 29513 + int(distinct), str(tmp_path), distinct),
                       nprocs=world, join=True,
                       start_method="spawn")
    got = [np.full_like(w, np.nan) for w in want]
    for r in range(world):
        z = np.load(tmp_path / f"s{r}.npz")
        for g, key in zip(got, ("x", "v", "F")):
            g[z["ids"]] = z[key]
    for g, w in zip(got, want):
        assert not np.isnan(g).any()
        np.testing.assert_allclose(g, w, rtol=1e-12, atol=1e-14 * np.abs(w).max())


def _nccl_rank(rank, world, port, out_dir, overlap):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SPHB_HALO_PUSH="0",
                      SPHB_SLAB_OVERLAP="1" if overlap else "0")
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        from paper_2405_05155_b200 import configs
        from paper_2405_05155_b200.eulerian import WEAKLY_COMPRESSIBLE, EosParams, FluidState
        from paper_2405_05155_b200.slab import slab_eulerian

        cfg = configs.c5_tgv3d(kernel="1.6h", n_side=24)
        n = cfg["pos"].shape[0]
        st = FluidState(cfg["vol"].copy(), cfg["rho"].copy(), cfg["mom"].copy(), None, n)
        s = slab_eulerian(cfg["pos"], st, EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0),
                          cfg["spec"], rank=rank, world=world, dist=dist,
                          cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
        assert (s._overlap is not None) == overlap
        s.advance(5)
        ids, rho, mom = s.owned()
        np.savez(os.path.join(out_dir, f"n{rank}.npz"), ids=ids, rho=rho, mom=mom)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (NCCL over NVLink)")
@pytest.mark.parametrize("overlap", [False, True])
def test_slab_nccl_two_gpus(tmp_path, overlap):
    """The torchrun path itself: two ranks on two GPUs with the NCCL halo
    exchange (boundary-first overlap on / off) equal the one-GPU solver."""
    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver,
                                                FluidState)

    cfg = configs.c5_tgv3d(kernel="1.6h", n_side=24)
    n = cfg["pos"].shape[0]
    ref = EulerianSolver(cfg["pos"], n, FluidState(cfg["vol"].copy(), cfg["rho"].copy(),
                                                   cfg["mom"].copy(), None, n),
                         EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0), cfg["spec"], None,
                         cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
    ref.advance(5)
    want = ref.state
    world = 2
    mp.start_processes(_nccl_rank, args=(world, 29521 + int(overlap), str(tmp_path), overlap),
                       nprocs=world, join=True, start_method="spawn")
    got_rho = np.full(n, np.nan)
    got_mom = np.full((n, 3), np.nan)
    for r in range(world):
        z = np.load(tmp_path / f"n{r}.npz")
        got_rho[z["ids"]] = z["rho"]
        got_mom[z["ids"]] = z["mom"]
    assert not np.isnan(got_rho).any()
    np.testing.assert_allclose(got_rho, want.rho, rtol=1e-14, atol=0)
    np.testing.assert_allclose(got_mom, want.mom, rtol=1e-12, atol=1e-14)


def _nccl_solid_rank(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SPHB_HALO_PUSH="0")
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        from paper_2405_05155_b200 import configs
        from paper_2405_05155_b200.slab import slab_solid

        cfg = configs.c4_column(kernel="1.6h", n_width=6)
        s = slab_solid(cfg["X0"], cfg["material"], cfg["spec"], cfg["dp"], rank=rank,
                       world=world, dist=dist, fixed=cfg["fixed"], cfl=cfg["cfl"])
        s.v = cfg["v0"][s.local_ids]
        s.advance(10)
        ids, x, v, F = s.owned()
        np.savez(os.path.join(out_dir, f"t{rank}.npz"), ids=ids, x=x, v=v, F=F)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (NCCL over NVLink)")
def test_slab_solid_nccl_two_gpus(tmp_path):
    """TL-SPH slab ranks on two GPUs with the NCCL exchange of Q, a and v."""
    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.tlsph import SolidSystem

    cfg = configs.c4_column(kernel="1.6h", n_width=6)
    ref = SolidSystem(cfg["X0"], cfg["material"], cfg["spec"], cfg["dp"], fixed=cfg["fixed"],
                      cfl=cfg["cfl"])
    ref.v = cfg["v0"]
    ref.advance(10)
    want = (ref.x, ref.v, ref.F)
    world = 2
    mp.start_processes(_nccl_solid_rank, args=(world, 29525, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    got = [np.full_like(w, np.nan) for w in want]
    for r in range(world):
        z = np.load(tmp_path / f"t{r}.npz")
        for g, key in zip(got, ("x", "v", "F")):
            g[z["ids"]] = z[key]
    for g, w in zip(got, want):
        assert not np.isnan(g).any()
        np.testing.assert_allclose(g, w, rtol=1e-12, atol=1e-14 * np.abs(w).max())
