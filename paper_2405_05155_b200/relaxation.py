"""Constant-pressure particle relaxation on the GPU (periodic boxes).

Drop-in for the hot-path part of `sph_trunc.relaxation` (reference
relaxation.py:1-210):

* `relax_accelerations(nlist, vols, spec, p0, rho0)` — the _pressure_accel
  loop (relaxation.py:66-89) over a device CSR (sphb_pressure_accel).
* `relax(config)` — the pseudo-time loop (relaxation.py:132-210) for
  `periodic_box` configs.  Each step bins the particles (sphb_bin) and runs
  the fused stencil-walk acceleration (sphb_relax_accel, no neighbour list is
  materialised) and the capped, wrapped update (sphb_relax_update).  The
  residual, best-state tracking and stop tests are the reference's.
* `relax_steps(...)` — the same loop with a fixed number of updates and no
  stop tests (the C1 benchmark protocol).
* shape-bounded relaxation: `relax(config)` without a
  periodic box runs `ShapeRelaxer` — open-domain binning from device-side
  bounds, the same fused acceleration, the analytic wall confinement
  (relaxation.py:92-117, 162-168; `wall_confinement`) and the capped update
  with surface projection (:120-129, 188-198), all in csrc/relax_shape.cu.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from .correction import _vols_dev
from .kernels import KernelSpec, kernel_spec, kernel_value
from .neighbors import NeighborList, make_grid


class RelaxationError(RuntimeError):
    """Raised when the residual diverges instead of settling."""


@dataclass
class RelaxationConfig:
    shape: object
    dp: float
    kernel: KernelSpec
    p0: float = 1.0
    step_scale: float = 0.2
    residual_tol: float = 2e-3
    max_steps: int = 1000
    rho0: float = 1.0
    patience: int | None = 250
    periodic_box: tuple | None = None

    def __post_init__(self):
        if self.p0 <= 0.0:
            raise ValueError("p0 must be positive")
        if not 0.0 < self.step_scale <= 0.5:
            raise ValueError("step_scale must lie in (0, 0.5]")
        if self.residual_tol <= 0.0:
            raise ValueError("residual_tol must be positive")


@dataclass
class RelaxResult:
    positions: np.ndarray
    residuals: np.ndarray
    steps: int
    converged: bool
    n_isolated: int
    best_step: int = 0
    best_residual: float = float("inf")


def relax_accelerations_device(nlist: NeighborList, vols, spec: KernelSpec, p0=1.0, rho0=1.0):
    torch = _lib.torch_cuda()
    starts, idx, r, e = nlist.device_csr()
    n, d = nlist.n, e.shape[1]
    acc = torch.empty((max(n, 1), d), dtype=torch.float64, device=starts.device)
    k = _lib.kernel_struct(spec)
    _lib.call("sphb_pressure_accel", n, d, starts.data_ptr(), idx.data_ptr(), r.data_ptr(),
              e.data_ptr(), _vols_dev(vols, n).data_ptr(), ctypes.byref(k), float(p0),
              float(rho0), acc.data_ptr(), _lib.stream_ptr())
    return acc[:n]


def relax_accelerations(nlist, vols, spec: KernelSpec, p0: float = 1.0, rho0: float = 1.0):
    """a_i = sum_j -2 p0 V_j grad W_ij / rho0; zero for isolated particles."""
    return relax_accelerations_device(nlist, vols, spec, p0, rho0).cpu().numpy()


@lru_cache(maxsize=None)
def _wall_kernel_table(family: str, h: float, dim: int, n_s: int = 256, n_t: int = 2000):
    """w2(s), the kernel integrated over the plane at offset s from the
    particle, on s in [0, kappa h] (relaxation.py:92-111): midpoint rule in
    the in-plane radius t over (0, kappa h)."""
    spec = kernel_spec(family, h, dim)
    cut = spec.kappa * h
    s = np.linspace(0.0, cut, n_s)
    if dim == 1:
        return s, kernel_value(spec, s)
    t = (np.arange(n_t) + 0.5) * (cut / n_t)
    w = kernel_value(spec, np.sqrt(s[:, None] ** 2 + t[None, :] ** 2))
    if dim == 3:
        w = 2.0 * np.pi * np.sum(w * t[None, :], axis=1) * (cut / n_t)
    else:
        w = 2.0 * np.sum(w, axis=1) * (cut / n_t)
    return s, w


def wall_confinement(spec: KernelSpec, depth) -> np.ndarray:
    """Inward acceleration magnitude per 2 p0 / rho at `depth` below the
    surface (relaxation.py:114-117): w2 interpolated, 0 beyond the support."""
    s_grid, w2 = _wall_kernel_table(spec.family, spec.h, spec.dim)
    return np.interp(np.asarray(depth, dtype=float), s_grid, w2, right=0.0)


class PeriodicRelaxer:
    """Device-resident relaxation state for a periodic box.

    Buffers are allocated once; `accelerate()` + `update()` are one step of
    relaxation.py:157-195 with no host synchronisation except reading the
    residual when the caller asks for it.
    """

    def __init__(self, positions, spec: KernelSpec, box, dp: float, *, p0=1.0, rho0=1.0,
                 step_scale=0.2, vols=None):
        torch = _lib.torch_cuda()
        pos = np.ascontiguousarray(np.asarray(positions, dtype=float))
        self.n, self.dim = pos.shape
        self.spec = spec
        self.box = np.asarray(box, dtype=float)
        self.p0, self.rho0 = float(p0), float(rho0)
        self.dt2 = step_scale * spec.h**2 * rho0 / p0          # relaxation.py:146
        self.cap = 0.25 * dp                                   # relaxation.py:147
        self.grid = make_grid(pos, spec.kappa * spec.h, self.box)
        self.kernel = _lib.kernel_struct(spec)
        dev = _lib.device()
        self.pos = _lib.to_device(pos, torch.float64)
        v = np.full(self.n, dp**self.dim) if vols is None else np.asarray(vols, dtype=float)
        self.vols = _lib.to_device(v, torch.float64)
        n1 = max(self.n, 1)
        self.ws = torch.empty((self.dim, n1), dtype=torch.float64, device=dev)
        self.perm = torch.empty(n1, dtype=torch.int32, device=dev)
        self.cs = torch.empty(self.grid.ntot, dtype=torch.int32, device=dev)
        self.ce = torch.empty(self.grid.ntot, dtype=torch.int32, device=dev)
        self.acc = torch.empty((n1, self.dim), dtype=torch.float64, device=dev)
        self.sums = torch.zeros(2, dtype=torch.float64, device=dev)
        self.wbytes = _lib.load_library().sphb_bin_workspace_bytes(self.n, ctypes.byref(self.grid))
        self.work = torch.empty(max(self.wbytes, 1), dtype=torch.uint8, device=dev)
        self._box3 = (ctypes.c_double * 3)(*(list(self.box) + [1.0] * (3 - self.dim)))
        self.launches_per_step = 0

    def accelerate(self):
        """Bin + fused acceleration; acc and {sum|a|, n_isolated} on the device."""
        s = _lib.stream_ptr()
        g = ctypes.byref(self.grid)
        _lib.call("sphb_bin", g, self.pos.data_ptr(), self.n, self.ws.data_ptr(),
                  self.perm.data_ptr(), self.cs.data_ptr(), self.ce.data_ptr(),
                  self.work.data_ptr(), self.wbytes, s)
        _lib.call("sphb_relax_accel", g, self.n, self.ws.data_ptr(), self.perm.data_ptr(),
                  self.cs.data_ptr(), self.ce.data_ptr(), self.vols.data_ptr(),
                  ctypes.byref(self.kernel), self.p0, self.rho0, self.acc.data_ptr(),
                  self.sums.data_ptr(), s)

    def residual(self) -> tuple[float, int]:
        """(mean|a| h rho0 / p0, n_isolated) of the last accelerate() (:170, :159)."""
        tot, iso = self.sums.tolist()
        mean = tot / self.n if self.n else float("nan")
        return float(mean * self.spec.h * self.rho0 / self.p0), int(iso)

    def update(self):
        """dx = a dt2, capped at 0.25 dp, pos = (pos + dx) % box (:188-195)."""
        _lib.call("sphb_relax_update", self.n, self.dim, self.acc.data_ptr(), self.dt2,
                  self.cap, self._box3, self.pos.data_ptr(), _lib.stream_ptr())

    def positions(self) -> np.ndarray:
        return self.pos[:self.n].cpu().numpy()

    def run(self, n_updates: int, *, graph: bool = True) -> None:
        """n_updates x (bin + fused acceleration + capped update), no host
        synchronisation; one update is captured as a CUDA graph (sort and
        memsets included) and replayed."""
        if n_updates <= 0:
            return
        if not graph:
            for _ in range(n_updates):
                self.accelerate()
                self.update()
            return
        torch = _lib.torch_cuda()
        from .eulerian import graph_steps

        per = graph_steps()          # updates per replay (amortises the replay latency)
        if getattr(self, "_graph", None) is None:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(per):
                    self.accelerate()
                    self.update()
            torch.cuda.synchronize()
            self._graph = g
        for _ in range(n_updates // per):
            self._graph.replay()
        for _ in range(n_updates % per):
            self.accelerate()
            self.update()


class ShapeRelaxer(PeriodicRelaxer):
    """Device-resident relaxation inside an SDF shape (open domain).

    Per step: device bounds -> cell grid (the reference's open-domain shift
    and extent, neighbors.py:194-203), bin, fused acceleration, wall
    confinement + |a| sum; update = capped move + surface projection.
    """

    def __init__(self, positions, spec: KernelSpec, shape, dp: float, *, p0=1.0, rho0=1.0,
                 step_scale=0.2, vols=None):
        torch = _lib.torch_cuda()
        pos = np.ascontiguousarray(np.asarray(positions, dtype=float))
        self.n, self.dim = pos.shape
        self.spec, self.shape = spec, shape
        self.sstruct = shape.device_struct()
        if self.sstruct.dim != self.dim:
            raise ValueError("shape and particle dimensions differ")
        self.p0, self.rho0 = float(p0), float(rho0)
        self.dt2 = step_scale * spec.h**2 * rho0 / p0          # relaxation.py:146
        self.cap = 0.25 * dp                                   # relaxation.py:147
        self.surf_tol = 1e-9 * dp                              # relaxation.py:148
        self.cutoff = spec.kappa * spec.h
        self.coef = 2.0 * p0 / rho0                            # relaxation.py:168
        self.kernel = _lib.kernel_struct(spec)
        dev = _lib.device()
        self._dev = dev
        self.pos = _lib.to_device(pos, torch.float64)
        v = np.full(self.n, dp**self.dim) if vols is None else np.asarray(vols, dtype=float)
        self.vols = _lib.to_device(v, torch.float64)
        n1 = max(self.n, 1)
        self.ws = torch.empty((self.dim, n1), dtype=torch.float64, device=dev)
        self.perm = torch.empty(n1, dtype=torch.int32, device=dev)
        self.acc = torch.empty((n1, self.dim), dtype=torch.float64, device=dev)
        self.sums = torch.zeros(3, dtype=torch.float64, device=dev)
        self.bounds = torch.empty(2 * self.dim, dtype=torch.float64, device=dev)
        s_grid, w2 = _wall_kernel_table(spec.family, spec.h, spec.dim)
        self.s_grid = _lib.to_device(np.ascontiguousarray(s_grid), torch.float64)
        self.w2 = _lib.to_device(np.ascontiguousarray(w2), torch.float64)
        self.n_s = int(s_grid.shape[0])
        self.cs = self.ce = self.work = None
        self._ntot = self._wcap = 0
        self.launches_per_step = 0

    def _grid(self):
        _lib.call("sphb_bounds", self.n, self.dim, self.pos.data_ptr(),
                  self.bounds.data_ptr(), _lib.stream_ptr())
        b = self.bounds.tolist()
        self.grid = make_grid(None, self.cutoff, None, dim=self.dim, lo=b[:self.dim],
                              hi=b[self.dim:])
        torch = _lib.torch_cuda()
        if self.grid.ntot > self._ntot:
            self._ntot = self.grid.ntot
            self.cs = torch.empty(self._ntot, dtype=torch.int32, device=self._dev)
            self.ce = torch.empty(self._ntot, dtype=torch.int32, device=self._dev)
        self.wbytes = _lib.load_library().sphb_bin_workspace_bytes(self.n, ctypes.byref(self.grid))
        if self.wbytes > self._wcap:
            self._wcap = max(self.wbytes, 1)
            self.work = torch.empty(self._wcap, dtype=torch.uint8, device=self._dev)

    def accelerate(self):
        """Bin (open grid) + fused acceleration + wall confinement."""
        self._grid()
        super().accelerate()
        _lib.call("sphb_relax_confine", ctypes.byref(self.sstruct), self.n, self.pos.data_ptr(),
                  self.cutoff, self.s_grid.data_ptr(), self.w2.data_ptr(), self.n_s, self.coef,
                  self.acc.data_ptr(), self.sums.data_ptr(), _lib.stream_ptr())

    def residual(self) -> tuple[float, int]:
        _, iso, tot = self.sums.tolist()
        mean = tot / self.n if self.n else float("nan")
        return float(mean * self.spec.h * self.rho0 / self.p0), int(iso)

    def update(self):
        _lib.call("sphb_relax_update_shape", ctypes.byref(self.sstruct), self.n,
                  self.acc.data_ptr(), self.dt2, self.cap, self.surf_tol, self.pos.data_ptr(),
                  _lib.stream_ptr())

    def run(self, n_updates: int, *, graph: bool = False) -> None:
        for _ in range(max(n_updates, 0)):     # the grid changes every step: no graph
            self.accelerate()
            self.update()


def relax_steps(positions, spec: KernelSpec, box, dp: float, n_updates: int, *, p0=1.0,
                rho0=1.0, step_scale=0.2, record_residuals=True):
    """`n_updates` relaxation updates from the given positions, no stop tests.

    Returns (positions after the last update, residuals of the n_updates + 1
    evaluations) — the C1 protocol of SURVEY Appendix B.
    """
    rl = PeriodicRelaxer(positions, spec, box, dp, p0=p0, rho0=rho0, step_scale=step_scale)
    residuals = []
    for step in range(n_updates + 1):
        rl.accelerate()
        if record_residuals:
            residuals.append(rl.residual()[0])
        if step < n_updates:
            rl.update()
    return rl.positions(), np.asarray(residuals)


def relax(config: RelaxationConfig) -> RelaxResult:
    """Drive a lattice fill to a low-residue distribution (relaxation.py:132-210):
    a periodic block when `periodic_box` is set, else the shape interior with
    wall confinement and surface projection."""
    from .geometry import lattice_fill

    spec = config.kernel
    pos0 = lattice_fill(config.shape, config.dp).copy()
    if config.periodic_box is not None:
        rl = PeriodicRelaxer(pos0, spec, config.periodic_box, config.dp, p0=config.p0,
                             rho0=config.rho0, step_scale=config.step_scale)
    else:
        rl = ShapeRelaxer(pos0, spec, config.shape, config.dp, p0=config.p0, rho0=config.rho0,
                          step_scale=config.step_scale)
    residuals: list[float] = []
    converged = False
    best_step, best_residual = 0, np.inf
    best_pos = rl.pos.clone()
    n_isolated = 0
    step = 0
    for step in range(config.max_steps + 1):
        rl.accelerate()
        residual, n_isolated = rl.residual()
        residuals.append(residual)
        if residual < best_residual:
            best_residual, best_step = residual, step
            best_pos.copy_(rl.pos)
        if residual < config.residual_tol:
            converged = True
            break
        if len(residuals) > 100 and residual > 10.0 * residuals[-101]:
            raise RelaxationError(
                f"relaxation residual diverged: {residuals[-101]:.3e} -> {residual:.3e}")
        if config.patience is not None and step - best_step >= config.patience:
            break
        if step == config.max_steps:
            break
        rl.update()
    final = rl.pos if converged else best_pos
    return RelaxResult(positions=final[:rl.n].cpu().numpy(), residuals=np.asarray(residuals),
                       steps=step, converged=converged, n_isolated=n_isolated,
                       best_step=best_step, best_residual=best_residual)
