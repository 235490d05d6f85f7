"""Multi-rank slab decomposition on CPU (gloo, world size 2 and 3).

Covers the host logic of the multi-GPU path (paper_2405_05155_b200/slab.py)
without a GPU: each rank builds its owned+halo particle set from the global
grid, runs the WC Eulerian step with the CPU oracle's loops on its local set,
exchanges halo layers with torch.distributed P2P (the exact calls the NCCL
path makes) and all-reduces the dt; rank 0 gathers the owned results and
compares them with a single-process run.  Because every owned row walks
exactly the global row in the global order, the result must be BIT-identical.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_05155_b200 import configs
from paper_2405_05155_b200.neighbors import make_grid
from paper_2405_05155_b200.slab import SlabPlan, cell_layer


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _flat_keys(pos, grid):
    d = pos.shape[1]
    key = np.zeros(pos.shape[0], dtype=np.int64)
    for a in range(d):
        key += cell_layer(pos, grid, a) * int(grid.strides[a])
    return key


def _oracle_rhs(nl, gwv, viscv, rho, mom, c, rho0, mu):
    from oracle import oracle as O

    p = np.ascontiguousarray(c**2 * (rho - rho0))
    v = np.ascontiguousarray(mom / rho[:, None])
    drho = np.empty(nl.n)
    dmom = np.zeros((nl.n, mom.shape[1]))
    O.lib().orc_rhs_wc(nl.n, mom.shape[1], O._p(nl.starts), O._p(nl.idx), O._p(nl.e), O._p(gwv),
                       O._p(viscv), O._p(np.ascontiguousarray(rho)), O._p(v), O._p(p), c, mu,
                       O._p(drho), O._p(dmom), None, None)
    return drho, dmom


def _geometry(pos, vol, spec, box, b):
    from oracle import oracle as O

    nl = O.build_neighbors(pos, spec.kappa * spec.h, box)
    gw = O.pair_gradients(nl, spec, b)
    gwv = np.ascontiguousarray(gw * vol[nl.idx][:, None])
    q = nl.r / spec.h
    dw = np.where(q <= spec.kappa, (spec.alpha / spec.h) * O._profile_deriv(spec.code, q), 0.0)
    return nl, gwv, np.ascontiguousarray(2.0 * dw / nl.r * vol[nl.idx])


def _run_rank(rank, world, port, n_side, steps, kernel, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O

        cfg = configs.c5_tgv3d(kernel=kernel, n_side=n_side)
        spec, box = cfg["spec"], cfg["box"]
        grid = make_grid(cfg["pos"], spec.kappa * spec.h, box)
        plan = SlabPlan(cfg["pos"], grid, rank, world)
        lpos = cfg["pos"][plan.local_ids]
        perm = np.argsort(_flat_keys(lpos, grid), kind="stable")   # the device binning order
        plan.attach(perm)
        gid = plan.local_ids[perm]                                 # sorted -> global id
        pos_s = cfg["pos"][gid]
        vol_s = cfg["vol"][gid]
        # B on the local set: exact for owned rows, then halo rows from owners
        nl = O.build_neighbors(pos_s, spec.kappa * spec.h, box)
        b = O.correction_matrices(nl, vol_s, spec)[0]
        bt = torch.from_numpy(np.ascontiguousarray(b))
        plan.exchange(dist, [bt])
        b = bt.numpy()
        nl, gwv, viscv = _geometry(pos_s, vol_s, spec, box, b)
        rho = torch.from_numpy(cfg["rho"][gid].copy())
        mom = torch.from_numpy(cfg["mom"][gid].copy())
        rows = plan.rows
        c, rho0, mu = cfg["c_art"], cfg["rho0"], cfg["mu"]
        for _ in range(steps):
            v = mom.numpy()[rows] / rho.numpy()[rows, None]
            smax = torch.tensor([float((c + np.linalg.norm(v, axis=1)).max())], dtype=torch.float64)
            dist.all_reduce(smax, op=dist.ReduceOp.MAX)
            dt = cfg["cfl"] * spec.h / float(smax)
            r0, m0 = rho.clone(), mom.clone()
            for frac in (0.5, 1.0):
                drho, dmom = _oracle_rhs(nl, gwv, viscv, rho.numpy(), mom.numpy(), c, rho0, mu)
                rho[rows] = r0[rows] + frac * dt * torch.from_numpy(drho[rows])
                mom[rows] = m0[rows] + frac * dt * torch.from_numpy(dmom[rows])
                plan.exchange(dist, [rho, mom])
        owned = torch.from_numpy(np.ascontiguousarray(gid[rows]))
        res = torch.cat([rho[rows, None], mom[rows]], dim=1)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([owned.numel()]))
        mx = int(max(s.item() for s in sizes))
        pad_ids = torch.full((mx,), -1, dtype=torch.int64)
        pad_ids[:owned.numel()] = owned
        pad_res = torch.zeros((mx, res.shape[1]), dtype=torch.float64)
        pad_res[:owned.numel()] = res
        all_ids = [torch.zeros_like(pad_ids) for _ in range(world)]
        all_res = [torch.zeros_like(pad_res) for _ in range(world)]
        dist.all_gather(all_ids, pad_ids)
        dist.all_gather(all_res, pad_res)
        if rank == 0:
            n = cfg["pos"].shape[0]
            full = np.full((n, res.shape[1]), np.nan)
            for ids, r in zip(all_ids, all_res):
                keep = ids >= 0
                full[ids[keep].numpy()] = r[keep].numpy()
            np.save(out, full)
    finally:
        dist.destroy_process_group()


def _single(n_side, steps, kernel):
    from oracle import oracle as O

    cfg = configs.c5_tgv3d(kernel=kernel, n_side=n_side)
    s = O.EulerianWC(cfg["pos"], cfg["vol"], cfg["rho"], cfg["mom"], cfg["spec"], cfg["c_art"],
                     cfg["rho0"], cfg["mu"], cfg["cfl"], cfg["box"])
    for _ in range(steps):
        s.step()
    return np.column_stack([s.rho, s.mom])


@pytest.mark.parametrize("world,kernel", [(2, "1.6h"), (3, "2h")])
def test_slab_wc_matches_single_rank_bitwise(tmp_path, world, kernel):
    n_side, steps = 16, 3
    out = str(tmp_path / "gathered.npy")
    mp.spawn(_run_rank, args=(world, _free_port(), n_side, steps, kernel, out), nprocs=world,
             join=True)
    got = np.load(out)
    want = _single(n_side, steps, kernel)
    assert not np.isnan(got).any()
    assert np.array_equal(got, want)


def test_slab_plan_layers_and_slices():
    cfg = configs.c5_tgv3d(n_side=16)
    spec = cfg["spec"]
    grid = make_grid(cfg["pos"], spec.kappa * spec.h, cfg["box"])
    world = 3
    owned_total = 0
    for rank in range(world):
        plan = SlabPlan(cfg["pos"], grid, rank, world)
        lpos = cfg["pos"][plan.local_ids]
        perm = np.argsort(_flat_keys(lpos, grid), kind="stable")
        plan.attach(perm)
        assert plan.rows.stop - plan.rows.start == plan.n_owned
        owned_total += plan.n_owned
        # halo slices are exactly the neighbours' boundary layers
        assert plan.recv_lo.stop - plan.recv_lo.start > 0
        assert plan.recv_hi.stop - plan.recv_hi.start > 0
    assert owned_total == cfg["pos"].shape[0]


def test_column_slabs_along_long_axis():
    """TL column: slabs along y (axis 1) with y as the storage slow axis;
    owned blocks and exchanged layers are contiguous and pair up."""
    cfg = configs.c4_column(n_width=6)
    spec = cfg["spec"]
    grid = make_grid(cfg["X0"], spec.kappa * spec.h, None, slow_axis=1)
    assert grid.sstrides[1] == grid.ncell[0] * grid.ncell[2]
    world = 4
    plans = []
    for rank in range(world):
        plan = SlabPlan(cfg["X0"], grid, rank, world)
        assert plan.axis == 1
        lpos = cfg["X0"][plan.local_ids]
        skey = sum(cell_layer(lpos, grid, a) * int(grid.sstrides[a]) for a in range(3))
        plan.attach(np.argsort(skey, kind="stable"))
        plans.append((plan, plan.local_ids[np.argsort(skey, kind="stable")]))
    # open ends: no lower halo on rank 0, no upper halo on the last rank
    assert plans[0][0].prev is None and plans[-1][0].next is None
    for (a, ga), (b, gb) in zip(plans[:-1], plans[1:]):
        assert np.array_equal(ga[a.send_hi], gb[b.recv_lo])   # a's last layer -> b's halo
        assert np.array_equal(gb[b.send_lo], ga[a.recv_hi])   # b's first layer -> a's halo
    assert sum(p.n_owned for p, _ in plans) == cfg["X0"].shape[0]


def test_slab_neighbor_rows_identical_to_global():
    from oracle import oracle as O

    cfg = configs.c5_tgv3d(n_side=16, kernel="2h")
    spec, box = cfg["spec"], cfg["box"]
    grid = make_grid(cfg["pos"], spec.kappa * spec.h, box)
    glob = O.build_neighbors(cfg["pos"], spec.kappa * spec.h, box)
    for rank in range(2):
        plan = SlabPlan(cfg["pos"], grid, rank, 2)
        lpos = cfg["pos"][plan.local_ids]
        perm = np.argsort(_flat_keys(lpos, grid), kind="stable")
        plan.attach(perm)
        gid = plan.local_ids[perm]
        loc = O.build_neighbors(cfg["pos"][gid], spec.kappa * spec.h, box)
        for s in range(plan.rows.start, plan.rows.stop, 97):
            i = gid[s]
            mine = gid[loc.idx[loc.starts[s]:loc.starts[s + 1]]]
            ref = glob.idx[glob.starts[i]:glob.starts[i + 1]]
            assert np.array_equal(mine, ref)
            assert np.array_equal(loc.r[loc.starts[s]:loc.starts[s + 1]],
                                  glob.r[glob.starts[i]:glob.starts[i + 1]])
