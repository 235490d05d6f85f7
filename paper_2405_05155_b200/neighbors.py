"""Cell-linked-list neighbour search on the GPU.

Drop-in for `sph_trunc.neighbors` (reference neighbors.py:1-241).

The reference bins particles into cells of edge >= cutoff with head/next
linked lists and walks the 3^d stencil twice (count, fill) on one CPU core
(neighbors.py:56-168).  Here the same grid (computed on the host exactly as
neighbors.py:183-203 does) is built on the device by
  sphb_bin        wrap/shift, cell key, stable radix sort, cell start/end
  sphb_csr_starts per-row counts + scan  -> CSR offsets
  sphb_csr_fill   idx, r, e
and the result is the reference's CSR, byte for byte: the same pairs, the
same row order, the same rounding of r and e.  It stays on the device; the
numpy views the reference API exposes (`starts`, `idx`, `r`, `e`) are
materialised on first access.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib


class NeighborList:
    """CSR neighbour list; e_ij = (x_i - x_j)/r points from j toward i.

    Same fields and helpers as the reference dataclass (neighbors.py:18-35).
    Arrays may live on the host (numpy) or on the device (torch); each side is
    produced from the other on demand.
    """

    def __init__(self, starts, idx, r, e, cutoff: float, bins: "CellBins | None" = None):
        self._host = {}
        self._dev = {}
        for name, arr in (("starts", starts), ("idx", idx), ("r", r), ("e", e)):
            if _is_tensor(arr):
                self._dev[name] = arr
            else:
                self._host[name] = np.asarray(arr)
        self.cutoff = float(cutoff)
        self.bins = bins

    # -- reference surface ---------------------------------------------------
    def _get(self, name):
        if name not in self._host:
            self._host[name] = self._dev[name].cpu().numpy()
        return self._host[name]

    @property
    def starts(self) -> np.ndarray:
        return self._get("starts")

    @property
    def idx(self) -> np.ndarray:
        return self._get("idx")

    @property
    def r(self) -> np.ndarray:
        return self._get("r")

    @property
    def e(self) -> np.ndarray:
        return self._get("e")

    @property
    def n(self) -> int:
        s = self._dev.get("starts")
        return (s.shape[0] if s is not None else self._host["starts"].shape[0]) - 1

    @property
    def m(self) -> int:
        s = self._dev.get("starts")
        return int(s[-1]) if s is not None else int(self._host["starts"][-1])

    @property
    def dim(self) -> int:
        e = self._dev.get("e")
        return (e if e is not None else self._host["e"]).shape[1]

    @property
    def counts(self) -> np.ndarray:
        return np.diff(self.starts)

    def neighbors_of(self, i: int) -> np.ndarray:
        return self.idx[self.starts[i]:self.starts[i + 1]]

    # -- device side ---------------------------------------------------------
    def device_csr(self):
        """(starts int64, idx int32, r f64, e f64[m, d]) as CUDA tensors."""
        torch = _lib.torch_cuda()
        for name, dt in (("starts", torch.int64), ("idx", torch.int32),
                         ("r", torch.float64), ("e", torch.float64)):
            if name not in self._dev:
                self._dev[name] = _lib.to_device(self._host[name], dt)
        return self._dev["starts"], self._dev["idx"], self._dev["r"], self._dev["e"]


def _is_tensor(a) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(a, torch.Tensor)


# ----------------------------------------------------------------- the grid
def make_grid(pos: np.ndarray | None, cutoff: float, box=None, *, dim: int | None = None,
              lo=None, hi=None, slow_axis: int | None = None) -> _lib.Grid:
    """Cell grid exactly as build_neighbors sets it up (neighbors.py:183-203).

    Either host positions, or (for device-resident sets) their per-axis
    min `lo` and max `hi`, give the open-domain shift and extent.
    """
    d = pos.shape[1] if pos is not None else int(dim)
    g = _lib.Grid()
    g.dim = d
    if box is not None:
        box_arr = np.asarray(box, dtype=float)
        lo_arr = np.zeros(d)
        extent = box_arr
        g.periodic = 1
    else:
        box_arr = np.ones(d)
        if pos is not None:
            lo_arr = pos.min(axis=0)
            wrapped_max = (pos - lo_arr).max(axis=0)
        else:
            lo_arr = np.asarray(lo, dtype=float)
            wrapped_max = np.asarray(hi, dtype=float) - lo_arr  # rounding is monotone
        extent = np.maximum(wrapped_max, cutoff)
        g.periodic = 0
    ncell = np.maximum((extent / cutoff).astype(np.int64), 1)
    inv_cell = ncell / box_arr if box is not None else np.full(d, 1.0 / cutoff)
    strides = np.ones(d, dtype=np.int64)
    for a in range(1, d):
        strides[a] = strides[a - 1] * ncell[a - 1]
    for a in range(3):
        g.ncell[a] = int(ncell[a]) if a < d else 1
        g.strides[a] = int(strides[a]) if a < d else 0
        g.inv_cell[a] = float(inv_cell[a]) if a < d else 0.0
        g.box[a] = float(box_arr[a]) if a < d else 1.0
        g.lo[a] = float(lo_arr[a]) if a < d else 0.0
    g.ntot = int(np.prod(ncell))
    # storage order: sort key with `slow_axis` slowest (default: the reference key)
    sa = d - 1 if slow_axis is None else int(slow_axis)
    if not 0 <= sa < d:
        raise ValueError("slow_axis out of range")
    g.slow_axis = sa
    order = [a for a in range(d) if a != sa] + [sa]
    st = 1
    for a in order:
        g.sstrides[a] = st
        st *= int(ncell[a])
    g.cutoff = float(cutoff)
    g.cut2 = float(cutoff) * float(cutoff)
    if g.ntot > 2**31 - 1:
        raise ValueError(f"cell grid too large ({g.ntot} cells); the domain is too sparse "
                         "for a uniform cell list at this cutoff")
    return g


class CellBins:
    """Particles binned on the device: sorted wrapped coordinates + cell tables."""

    def __init__(self, grid: _lib.Grid, n: int, ws, perm, cell_start, cell_end):
        self.grid = grid
        self.n = n
        self.dim = grid.dim
        self.ws = ws                  # (dim, n) float64, sorted SoA
        self.perm = perm              # (n,) int32 sorted -> original
        self.cell_start = cell_start  # (ntot,) int32
        self.cell_end = cell_end

    def rank(self):
        """(n,) int64 original -> sorted position."""
        torch = _lib.torch_cuda()
        r = torch.empty(self.n, dtype=torch.int64, device=self.perm.device)
        r[self.perm.long()] = torch.arange(self.n, device=self.perm.device)
        return r


def bin_particles(pos_dev, grid: _lib.Grid) -> CellBins:
    """sphb_bin on a (n, d) float64 CUDA tensor (orig order)."""
    torch = _lib.torch_cuda()
    n = pos_dev.shape[0]
    dev = pos_dev.device
    ws = torch.empty((grid.dim, max(n, 1)), dtype=torch.float64, device=dev)
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    cs = torch.empty(grid.ntot, dtype=torch.int32, device=dev)
    ce = torch.empty(grid.ntot, dtype=torch.int32, device=dev)
    nbytes = _lib.load_library().sphb_bin_workspace_bytes(n, C_ref(grid))
    work = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    _lib.call("sphb_bin", C_ref(grid), pos_dev.data_ptr(), n, ws.data_ptr(), perm.data_ptr(),
              cs.data_ptr(), ce.data_ptr(), work.data_ptr(), nbytes, _lib.stream_ptr())
    return CellBins(grid, n, ws[:, :n], perm[:n], cs, ce)


def C_ref(s):
    import ctypes

    return ctypes.byref(s)


def csr_from_bins(bins: CellBins):
    """Reference-order CSR (starts, idx, r, e) on the device from binned particles."""
    torch = _lib.torch_cuda()
    n, d = bins.n, bins.dim
    dev = bins.perm.device
    starts = torch.empty(n + 1, dtype=torch.int64, device=dev)
    nbytes = _lib.load_library().sphb_csr_workspace_bytes(n)
    work = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    ws = bins.ws.contiguous() if n else bins.ws
    _lib.call("sphb_csr_starts", C_ref(bins.grid), n, ws.data_ptr(), bins.perm.data_ptr(),
              bins.cell_start.data_ptr(), bins.cell_end.data_ptr(), starts.data_ptr(),
              work.data_ptr(), nbytes, _lib.stream_ptr())
    m = int(starts[-1].item())
    idx = torch.empty(m, dtype=torch.int32, device=dev)
    r = torch.empty(m, dtype=torch.float64, device=dev)
    e = torch.empty((m, d), dtype=torch.float64, device=dev)
    if m:
        _lib.call("sphb_csr_fill", C_ref(bins.grid), n, ws.data_ptr(), bins.perm.data_ptr(),
                  bins.cell_start.data_ptr(), bins.cell_end.data_ptr(), starts.data_ptr(),
                  idx.data_ptr(), r.data_ptr(), e.data_ptr(), _lib.stream_ptr())
    return starts, idx, r, e


def ell_from_bins(bins: CellBins, h: float, kappa: float):
    """Engine pass list in sorted space: (nbr [width, n] int32, cnt [n] int32, width).

    Same enumeration order as the CSR row, with the pairs every pass skips
    (q = r/h > kappa) dropped once here instead of tested in every pass.
    """
    torch = _lib.torch_cuda()
    n = bins.n
    dev = bins.perm.device
    cnt = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    mx = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = bins.ws.contiguous()
    _lib.call("sphb_ell_count", C_ref(bins.grid), n, ws.data_ptr(), bins.cell_start.data_ptr(),
              bins.cell_end.data_ptr(), float(h), float(kappa), cnt.data_ptr(), mx.data_ptr(),
              _lib.stream_ptr())
    width = int(mx.item())
    nbr = torch.empty((max(width, 1), max(n, 1)), dtype=torch.int32, device=dev)
    if width and n:
        _lib.call("sphb_ell_fill", C_ref(bins.grid), n, ws.data_ptr(), bins.cell_start.data_ptr(),
                  bins.cell_end.data_ptr(), float(h), float(kappa), width, nbr.data_ptr(),
                  _lib.stream_ptr())
    return nbr, cnt[:n], width


class EngineOrder:
    """Storage order of the stage engines (a layout choice, no reference
    counterpart): particles sorted by a lattice-spacing key (slow axis
    slowest, axis 0 fastest) instead of by cell, so that on lattices
    consecutive rows are consecutive lattice sites.  Same fields as CellBins
    where the engines read them; `q` maps engine position -> cell-sorted
    position for per-particle arrays built in cell order."""

    def __init__(self, grid, n, ws, perm, q):
        self.grid, self.n, self.dim = grid, n, grid.dim
        self.ws, self.perm, self.q = ws, perm, q

    def rank(self):
        torch = _lib.torch_cuda()
        r = torch.empty(self.n, dtype=torch.int64, device=self.perm.device)
        r[self.perm.long()] = torch.arange(self.n, device=self.perm.device)
        return r


def engine_order(bins: CellBins, nbr, cnt, width: int, spacing: float | None = None,
                 tile=None):
    """Re-store binned particles in lattice order and remap their ELL list.

    The rows are then sorted by quantised displacement (sphb_ell_sort_rows),
    so on a lattice every row lists the same offsets in the same order and
    the lanes of a warp gather consecutive records.  The pair sets are
    unchanged; only storage and summation order differ.  Returns
    (EngineOrder, nbr, cnt).
    """
    torch = _lib.torch_cuda()
    n, d, g = bins.n, bins.dim, bins.grid
    dev = bins.perm.device
    ws = bins.ws
    if n == 0:
        return EngineOrder(g, n, ws, bins.perm, torch.zeros(0, dtype=torch.int64, device=dev)), \
            nbr, cnt
    if spacing is None:            # mean spacing of the set
        ext = ([g.box[a] for a in range(d)] if g.periodic
               else [max(float(ws[a].max().item()), 1e-300) for a in range(d)])
        spacing = float(np.prod(ext) / n) ** (1.0 / d)
    # lattice key: a periodic lattice sits at cell centres ((k + 1/2) spacing
    # of the wrapped coordinate); an open one starts at 0 (w = x - min, a
    # multiple of the spacing up to rounding), so round instead of floor
    shift = 0.0 if g.periodic else 0.5
    k = torch.floor(ws * (1.0 / spacing) + shift).to(torch.int64).clamp_(min=0)
    tile = tuple(tile or ()) + (1,) * (d - len(tile or ()))
    # slowest component: the cell layer along the grid's storage slow axis
    # (as the binning computes it), so a slab rank's owned block and halo
    # layers stay contiguous; then tiles of tile[0] x tile[1] x ... sites in
    # lattice order, sites inside a tile in lattice order; the slow axis is
    # the slowest lattice axis, axis 0 (or the next) the fastest
    sa = int(g.slow_axis)
    axes = [sa] + [a for a in range(d - 1, -1, -1) if a != sa]
    layer = torch.floor(ws[sa] * g.inv_cell[sa]).to(torch.int64)
    layer = (torch.remainder(layer, int(g.ncell[sa])) if g.periodic
             else layer.clamp(0, int(g.ncell[sa]) - 1))
    kt = torch.stack([k[a] // tile[a] for a in range(d)])
    kr = torch.stack([k[a] % tile[a] for a in range(d)])
    top = kt.max(dim=1).values + 1
    key = layer.clone()
    for a in axes:
        key = key * top[a] + kt[a]
    for a in axes:
        key = key * tile[a] + kr[a]
    q = torch.sort(key, stable=True).indices
    qinv = torch.empty(n, dtype=torch.int64, device=dev)
    qinv[q] = torch.arange(n, device=dev)
    cnt_e = cnt[q].contiguous()
    nbr_e = torch.zeros_like(nbr)
    for r in range(width):
        col = nbr[r, q].long()
        ok = cnt_e > r
        nbr_e[r] = torch.where(ok, qinv[torch.where(ok, col, 0)], 0).to(torch.int32)
    ws_e = ws[:, q].contiguous()
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("sphb_ell_sort_rows", C_ref(g), n, ws_e.data_ptr(), nbr_e.data_ptr(),
              cnt_e.data_ptr(), float(spacing), err.data_ptr(), _lib.stream_ptr())
    if int(err.item()):
        return EngineOrder(g, n, ws, bins.perm, torch.arange(n, device=dev)), nbr, cnt
    return EngineOrder(g, n, ws_e, bins.perm[q].contiguous(), q), nbr_e, cnt_e


# ---------------------------------------------------------- reference API
def _validate(positions, cutoff, box):
    """Input checks of build_neighbors (neighbors.py:173-188)."""
    pos = np.ascontiguousarray(np.asarray(positions, dtype=float))
    if pos.ndim != 2:
        raise ValueError("positions must have shape (n, dim)")
    if not np.all(np.isfinite(pos)):
        raise ValueError("positions must be finite")
    if not (cutoff > 0.0 and np.isfinite(cutoff)):
        raise ValueError("cutoff must be positive and finite")
    if box is not None:
        box_arr = np.asarray(box, dtype=float)
        if box_arr.shape != (pos.shape[1],) or np.any(box_arr <= 0.0):
            raise ValueError("periodic box must give a positive length per axis")
        if np.any(box_arr < 2.0 * cutoff):
            raise ValueError("periodic box must be at least two cutoffs wide")
    return pos


def build_neighbors(positions, cutoff: float, box=None) -> NeighborList:
    """All pairs with 0 < r_ij <= cutoff; minimum image when a box is given."""
    pos = _validate(positions, cutoff, box)
    grid = make_grid(pos, cutoff, box)
    pos_dev = _lib.to_device(pos, _lib.torch_cuda().float64)
    bins = bin_particles(pos_dev, grid)
    starts, idx, r, e = csr_from_bins(bins)
    return NeighborList(starts, idx, r, e, cutoff=float(cutoff), bins=bins)


def interior_mask(positions, margin: float) -> np.ndarray:
    """Particles at least `margin` inside the bounding box (neighbors.py:403-408)."""
    pos = np.asarray(positions, dtype=float)
    lo = pos.min(axis=0)
    hi = pos.max(axis=0)
    return np.all((pos >= lo + margin) & (pos <= hi - margin), axis=1)


def neighbor_count_ratio(positions, cutoff_tw: float, cutoff_sw: float) -> float:
    """Mean truncated over mean standard neighbour count, interior particles
    only (neighbors.py:411-431)."""
    pos = np.asarray(positions, dtype=float)
    if pos.size == 0:
        raise ValueError("empty particle set")
    if not (cutoff_tw > 0.0 and cutoff_sw > 0.0):
        raise ValueError("cutoffs must be positive")
    inner = interior_mask(pos, cutoff_sw)
    if not np.any(inner):
        raise ValueError("no interior particles at this cutoff")
    mean_tw = build_neighbors(pos, cutoff_tw).counts[inner].mean()
    mean_sw = build_neighbors(pos, cutoff_sw).counts[inner].mean()
    if mean_sw == 0.0:
        raise ValueError("standard-cutoff neighborhoods are empty")
    return float(mean_tw / mean_sw)
