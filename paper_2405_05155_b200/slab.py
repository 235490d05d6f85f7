"""Slab domain decomposition of a static particle set over GPUs.

The reference runs on one core (no parallelism at all); this is
the one parallel strategy the B200 design adds.  Particles are
fixed in both solvers, so the decomposition is static:

* the GLOBAL cell grid (neighbors.py:183-203 set-up on all particles) is cut
  into slabs of whole cell layers along the slowest flat-key axis (the last
  axis: z in 3D), rank r owning layers [z0, z1);
* a rank holds its owned particles plus one halo cell layer on each side
  (cell edge >= cutoff, so every neighbour of an owned particle is there),
  listed in ascending global index and binned with the global grid, so rows
  enumerate exactly the global neighbour set in the reference's order;
* because z is the slowest key axis, in cell-sorted order the owned
  particles form one contiguous block and every exchanged layer is a
  contiguous slice: the halo exchange sends/receives slices of the state
  records in place (no pack/unpack kernels).

Exchange pattern per WC stage (and once at set-up for B): send the first
owned layer to the previous rank and the last owned layer to the next rank;
receive the halo layers from them (periodic ring for TGV, open ends for a
column).  Messages are issued in a fixed order (to-next before to-prev,
from-prev before from-next) so the k-th send from a rank pairs with the k-th
receive on its peer even when prev == next (world size 2).

Host-side logic only in this module; it runs unchanged with the gloo
backend on CPU tensors (tests/test_slab_cpu.py) and with NCCL on device
buffers (EulerianSolver(_slab=...)).
"""

from __future__ import annotations

import numpy as np


def cell_layer(pos: np.ndarray, grid, axis: int) -> np.ndarray:
    """Cell coordinate along `axis` exactly as _cell_index computes it
    (neighbors.py:38-53 on the coordinates of neighbors.py:189/194)."""
    x = np.asarray(pos, dtype=float)[:, axis]
    if grid.periodic:
        w = np.remainder(x, grid.box[axis])
    else:
        w = x - grid.lo[axis]
    c = np.floor(w * grid.inv_cell[axis]).astype(np.int64)
    n = int(grid.ncell[axis])
    if grid.periodic:
        return np.mod(c, n)
    return np.clip(c, 0, n - 1)


class SlabPlan:
    """Owned/halo particle sets of one rank and its exchange slices."""

    def __init__(self, positions, grid, rank: int, world: int, axis: int | None = None):
        pos = np.asarray(positions, dtype=float)
        self.dim = pos.shape[1]
        self.axis = int(grid.slow_axis) if axis is None else axis
        if self.axis != grid.slow_axis:
            raise ValueError("slabs are cut along the grid's storage slow axis")
        self.rank, self.world = int(rank), int(world)
        self.periodic = bool(grid.periodic)
        nz = int(grid.ncell[self.axis])
        self.nz = nz
        if world > 1 and nz < 2 * world:
            raise ValueError(f"{nz} cell layers cannot be cut into {world} slabs of >= 2 layers")
        self.z0 = rank * nz // world
        self.z1 = (rank + 1) * nz // world
        layer = cell_layer(pos, grid, self.axis)
        self.layer_all = layer
        owned = (layer >= self.z0) & (layer < self.z1)
        self.lo_halo = self.hi_halo = None
        self.prev = self.next = None
        if world > 1:
            if self.periodic or rank > 0:
                self.lo_halo = (self.z0 - 1) % nz
                self.prev = (rank - 1) % world
            if self.periodic or rank < world - 1:
                self.hi_halo = self.z1 % nz
                self.next = (rank + 1) % world
        halo = np.zeros_like(owned)
        for h in (self.lo_halo, self.hi_halo):
            if h is not None:
                halo |= layer == h
        self.local_ids = np.nonzero(owned | halo)[0]      # ascending global index
        self.owned_ids = np.nonzero(owned)[0]
        self.local_layer = layer[self.local_ids]
        self.n_local = self.local_ids.size
        self.n_owned = self.owned_ids.size

    def attach(self, perm_sorted_to_local: np.ndarray) -> None:
        """Contiguous sorted-order slices, given the device binning's perm."""
        lay = self.local_layer[np.asarray(perm_sorted_to_local, dtype=np.int64)]
        self.sorted_layer = lay

        def block(mask, what):
            idx = np.nonzero(mask)[0]
            if idx.size == 0:
                return slice(0, 0)
            if idx[-1] - idx[0] + 1 != idx.size:
                raise RuntimeError(f"{what} is not contiguous in cell-sorted order")
            return slice(int(idx[0]), int(idx[-1]) + 1)

        self.rows = block((lay >= self.z0) & (lay < self.z1), "owned block")
        self.send_lo = block(lay == self.z0, "first owned layer")
        self.send_hi = block(lay == self.z1 - 1, "last owned layer")
        self.recv_lo = block(lay == self.lo_halo, "lower halo") if self.lo_halo is not None else None
        self.recv_hi = block(lay == self.hi_halo, "upper halo") if self.hi_halo is not None else None

    def p2p_ops(self, dist, bufs, group=None):
        """P2POp list exchanging the halo slices of every tensor in `bufs`
        (each indexed by sorted particle along dim 0)."""
        ops = []
        for buf in bufs:
            if self.next is not None:
                ops.append(dist.P2POp(dist.isend, buf[self.send_hi], self.next, group))
            if self.prev is not None:
                ops.append(dist.P2POp(dist.isend, buf[self.send_lo], self.prev, group))
            if self.prev is not None:
                ops.append(dist.P2POp(dist.irecv, buf[self.recv_lo], self.prev, group))
            if self.next is not None:
                ops.append(dist.P2POp(dist.irecv, buf[self.recv_hi], self.next, group))
        return ops

    def share_buffers(self, dist, tensors):
        """Peer pointers for the fused halo push (sphb_wc_params.push_*).

        Every rank passes its record buffers in the same order; returns
        {"prev": ([ptr per buffer], halo_start), "next": (...)} with the
        neighbour ranks' device addresses of those buffers and the record
        index of the halo slice this rank fills (prev: its upper halo, next:
        its lower halo).  Thread ranks (tests) share raw pointers through
        `dist.share_device_buffers`; torch.distributed ranks exchange CUDA IPC
        handles of the storages (all_gather_object) and map them here.
        """
        halo = (self.recv_lo.start if self.recv_lo is not None else -1,
                self.recv_hi.start if self.recv_hi is not None else -1)
        if hasattr(dist, "share_device_buffers"):
            table = dist.share_device_buffers([t.data_ptr() for t in tensors], halo)
        else:
            import torch

            mine = ([(t.untyped_storage()._share_cuda_(), t.storage_offset() * t.element_size())
                     for t in tensors], halo)
            allinfo = [None] * self.world
            dist.all_gather_object(allinfo, mine)
            table = {}
            self._ipc_keep = []
            for r in {self.prev, self.next} - {None}:
                ptrs = []
                for handle, off in allinfo[r][0]:
                    st = torch.UntypedStorage._new_shared_cuda(*handle)
                    self._ipc_keep.append(st)
                    ptrs.append(st.data_ptr() + off)
                table[r] = (ptrs, allinfo[r][1])
        out = {}
        if self.prev is not None:
            out["prev"] = (table[self.prev][0], table[self.prev][1][1])   # its upper halo
        if self.next is not None:
            out["next"] = (table[self.next][0], table[self.next][1][0])   # its lower halo
        return out

    def exchange(self, dist, bufs, group=None, reuse: bool = False) -> None:
        """Blocking (host) / stream-ordered (NCCL) halo exchange of `bufs`.

        reuse: the buffers are the solver's static record buffers (the step
        loop), so their P2POp list is built once and kept (it holds the
        views); per-step host work is then the batched launch itself."""
        if self.world == 1:
            return
        if reuse:
            cache = self.__dict__.setdefault("_ops_cache", {})
            key = (id(dist), id(group)) + tuple((b.data_ptr(), tuple(b.shape)) for b in bufs)
            ops = cache.get(key)
            if ops is None:
                ops = cache[key] = self.p2p_ops(dist, bufs, group)
        else:
            ops = self.p2p_ops(dist, bufs, group)
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()


def slab_eulerian(positions, state, eos, kernel, *, rank: int, world: int, dist,
                  correction: bool = True, cfl: float = 0.5, mu: float = 0.0,
                  periodic_box=None):
    """EulerianSolver for this rank's slab of a global particle set.

    `positions` / `state` are the GLOBAL inputs (every rank passes the same
    arrays); the solver holds owned + halo particles, updates the owned block
    and exchanges halo layers after every stage over `dist` (NCCL on GPUs).
    """
    from .eulerian import EulerianSolver, FluidState
    from .neighbors import make_grid

    pos = np.ascontiguousarray(positions, dtype=float)
    grid = make_grid(pos, kernel.kappa * kernel.h, periodic_box)
    plan = SlabPlan(pos, grid, rank, world)
    ids = plan.local_ids
    local = FluidState(vol=np.asarray(state.vol)[ids], rho=np.asarray(state.rho)[ids],
                       mom=np.asarray(state.mom)[ids], etot=None, n_interior=ids.size)
    return EulerianSolver(pos[ids], ids.size, local, eos, kernel, None, correction=correction,
                          cfl=cfl, mu=mu, periodic_box=periodic_box, _slab=plan, _grid=grid,
                          _dist=dist)


def slab_solid(X0, material, kernel, dp, *, rank: int, world: int, dist, fixed=None,
               correction: bool = True, cfl: float = 0.6, axis: int | None = None):
    """SolidSystem for this rank's slab of a global reference configuration.

    The slab axis defaults to the one with the most cell layers (the long
    axis of a column); particles are stored with that axis slowest so the
    owned block and the exchanged layers are contiguous.  Per step the halo
    receives Q after pass A and (v, a) after pass B.  Set the initial
    velocity with `system.v = v0[system.local_ids]`.
    """
    from .neighbors import make_grid
    from .tlsph import SolidSystem

    X = np.ascontiguousarray(X0, dtype=float)
    cut = kernel.kappa * kernel.h
    if axis is None:
        probe = make_grid(X, cut, None)
        axis = int(np.argmax([probe.ncell[a] for a in range(X.shape[1])]))
    grid = make_grid(X, cut, None, slow_axis=axis)
    plan = SlabPlan(X, grid, rank, world)
    ids = plan.local_ids
    fx = None if fixed is None else np.asarray(fixed, dtype=bool)[ids]
    system = SolidSystem(X[ids], material, kernel, dp, fixed=fx, correction=correction, cfl=cfl,
                         _slab=plan, _grid=grid, _dist=dist)
    system.local_ids = ids
    return system
