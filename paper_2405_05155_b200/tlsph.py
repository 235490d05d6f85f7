"""Total-Lagrangian SPH for elastic solids, on the GPU.

Drop-in for `sph_trunc.tlsph` (reference tlsph.py:1-254): `Material`,
`lame_params`, `pk2_stress`, `init_case_velocity`, `SolidStateError` and
`SolidSystem` with the reference constructor and `accelerations()`,
`deformation_rates()`, `stable_dt()`, `step(dt=None)`.

Engine (csrc/tl_engine.cu).  Construction bins the reference configuration
X0 once, builds the ELL pass list and B0 on the device.  A kick-drift-kick
step (tlsph.py:182-206) is three launches:
  sphb_set_dt     dt = cfl h / (c_s + max|v|)             (tlsph.py:178-180)
  sphb_tl_pass_a  half kick, drift, dF, F update, det check, Q = P B0^T
  sphb_tl_pass_b  momentum sum, second half kick, max|v| for the next dt
The reference-configuration gradients g0 = grad0 W V0 (tlsph.py:145-146)
are recomputed per pair from X0 instead of being streamed.

The constitutive law is St. Venant-Kirchhoff, the one the reference
implements (tlsph.py:54-65); BASELINE.json's "Neo-Hookean" has no reference
counterpart.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .kernels import CODE_WENDLAND, KernelSpec
from .neighbors import (NeighborList, bin_particles, csr_from_bins, ell_from_bins, engine_order,
                        make_grid)


class SolidStateError(RuntimeError):
    """Raised when the deformation gradient loses invertibility."""


def lame_params(E: float, nu: float) -> tuple[float, float]:
    """(lambda, G) from Young's modulus and Poisson ratio (tlsph.py:27-35)."""
    if not E > 0.0:
        raise ValueError("Young's modulus must be positive")
    if not -1.0 < nu < 0.5:
        raise ValueError("Poisson ratio must lie in (-1, 0.5); 0.5 makes lambda singular")
    return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


SVK = "svk"
NEO_HOOKEAN = "neo-hookean"
LAWS = {SVK: 0, NEO_HOOKEAN: 1}


@dataclass(frozen=True)
class Material:
    """Elastic material (tlsph.py:27-51).  `law` is an extension: the
    reference implements St. Venant-Kirchhoff only; "neo-hookean" selects
    the compressible Neo-Hookean law BASELINE's configs 3-4 name
    (S = G (I - C^-1) + lam ln(J) C^-1; not reference-backed)."""

    rho0: float
    E: float
    nu: float
    law: str = SVK

    def __post_init__(self):
        if self.law not in LAWS:
            raise ValueError(f"unknown material law {self.law!r}; expected one of {tuple(LAWS)}")

    @property
    def lame(self) -> tuple[float, float]:
        return lame_params(self.E, self.nu)

    @property
    def sound_speed(self) -> float:
        lam, g = self.lame
        return float(np.sqrt((lam + 2.0 * g) / self.rho0))


def pk2_stress(F, material: Material):
    """Second Piola-Kirchhoff stress: SVK lam tr(E) I + 2 G E
    (tlsph.py:54-65), or the compressible Neo-Hookean law of `material`."""
    F = np.asarray(F, dtype=float)
    lam, g = material.lame
    batch = F if F.ndim == 3 else F[None]
    eye = np.eye(batch.shape[-1])
    C = np.einsum("nba,nbc->nac", batch, batch)
    if getattr(material, "law", SVK) == NEO_HOOKEAN:
        ci = np.linalg.inv(C)
        ln_j = 0.5 * np.log(np.linalg.det(C))
        s = g * (eye - ci) + lam * ln_j[:, None, None] * ci
    else:
        strain = 0.5 * (C - eye)
        tr = np.trace(strain, axis1=1, axis2=2)
        s = lam * tr[:, None, None] * eye + 2.0 * g * strain
    return s if F.ndim == 3 else s[0]


TWIST = "twist"
BEND = "bend"


def von_mises(F, S):
    """Von Mises stress of the Cauchy stress J^-1 F S F^T (tlsph.py:68-86);
    2D tensors are read as plane stress (sigma_zz = 0).  Host diagnostic."""
    F = np.asarray(F, dtype=float)
    S = np.asarray(S, dtype=float)
    single = F.ndim == 2
    Fb, Sb = (F[None], S[None]) if single else (F, S)
    sigma = np.einsum("nab,nbc,ndc->nad", Fb, Sb, Fb) / np.linalg.det(Fb)[:, None, None]
    if sigma.shape[-1] == 2:
        pad = np.zeros((sigma.shape[0], 3, 3))
        pad[:, :2, :2] = sigma
        sigma = pad
    dev = sigma - (np.trace(sigma, axis1=1, axis2=2) / 3.0)[:, None, None] * np.eye(3)
    vm = np.sqrt(1.5 * np.einsum("nab,nab->n", dev, dev))
    return float(vm[0]) if single else vm


def init_case_velocity(kind: str, X0, *, length: float, omega0: float = 105.0,
                       v0=(10.0 * np.sqrt(3.0) / 2.0, 5.0, 0.0), axis_center=(0.0, 0.0)):
    """Column initial velocities (tlsph.py:233-254): twist = omega0 sin(pi y /
    (2L)) about the y axis; bend = uniform translation."""
    X0 = np.asarray(X0, dtype=float)
    if kind == BEND:
        return np.tile(np.asarray(v0, dtype=float)[:X0.shape[1]], (X0.shape[0], 1))
    if kind != TWIST:
        raise ValueError(f"unknown case kind {kind!r}")
    if X0.shape[1] != 3:
        raise ValueError("twist initial condition is three-dimensional")
    w = omega0 * np.sin(0.5 * np.pi * X0[:, 1] / length)
    v = np.zeros_like(X0)
    v[:, 0] = w * (X0[:, 2] - axis_center[1])
    v[:, 2] = -w * (X0[:, 0] - axis_center[0])
    return v


def _vec_rec(arr_sorted, n, dim, dev):
    torch = _lib.torch_cuda()
    out = torch.zeros((n, 4), dtype=torch.float64, device=dev)
    out[:, :dim] = arr_sorted
    return out


def _mat_rec(m_sorted, n, dim, dev):
    """(n, d, d) -> one record per particle (2D: {a00, a01, a10, a11};
    1D: {a00}); 3D matrices use _f_rec / _b0_rec / the Q planes."""
    torch = _lib.torch_cuda()
    assert dim < 3
    out = torch.zeros((n, 4), dtype=torch.float64, device=dev)
    out[:, :dim * dim] = m_sorted.reshape(n, dim * dim)
    return out


def _f_rec(m_sorted, n, dim, dev):
    """(n, d, d) -> deformation-gradient records (3D: 9 doubles in planes
    {F00,F01,F02,F10} {F11,F12,F20,F21} {F22}, tl_engine.cu load_f)."""
    if dim != 3:
        return _mat_rec(m_sorted, n, dim, dev)
    torch = _lib.torch_cuda()
    flat = m_sorted.reshape(n, 9)
    out = torch.empty(9 * n, dtype=torch.float64, device=dev)
    out[:4 * n].view(n, 4).copy_(flat[:, 0:4])
    out[4 * n:8 * n].view(n, 4).copy_(flat[:, 4:8])
    out[8 * n:].copy_(flat[:, 8])
    return out


def _f_unrec(rec, n_all, dim, rows=None):
    """F records -> (n, d, d) (optionally only `rows`)."""
    if dim != 3:
        return _mat_unrec(rec, n_all, dim, rows)
    rows = slice(0, n_all) if rows is None else rows
    torch = _lib.torch_cuda()
    p0 = rec[:4 * n_all].view(n_all, 4)[rows]
    p1 = rec[4 * n_all:8 * n_all].view(n_all, 4)[rows]
    p2 = rec[8 * n_all:][rows]
    return torch.cat([p0, p1, p2[:, None]], dim=1).reshape(-1, 3, 3)


def _b0_rec(b_sorted, n, dim, dev):
    """(n, d, d) symmetric B0 -> records (3D: planes {b00,b01,b02,b11} and
    {b12,b22}, symmetrised, tl_engine.cu load_b0)."""
    if dim != 3:
        return _mat_rec(b_sorted, n, dim, dev)
    torch = _lib.torch_cuda()
    bs = 0.5 * (b_sorted + b_sorted.transpose(1, 2))
    out = torch.empty(6 * n, dtype=torch.float64, device=dev)
    p0 = out[:4 * n].view(n, 4)
    p1 = out[4 * n:].view(n, 2)
    p0[:, 0], p0[:, 1], p0[:, 2], p0[:, 3] = bs[:, 0, 0], bs[:, 0, 1], bs[:, 0, 2], bs[:, 1, 1]
    p1[:, 0], p1[:, 1] = bs[:, 1, 2], bs[:, 2, 2]
    return out


def _mat_unrec(rec, n, dim, rows=None):
    """2D / 1D records -> (n, d, d) matrices (optionally only `rows`)."""
    assert dim < 3
    out = rec if rows is None else rec[rows]
    return out[:, :dim * dim].reshape(-1, dim, dim)


class SolidSystem:
    """Reference configuration, state and fused passes for one solid body."""

    def __init__(self, X0, material: Material, kernel: KernelSpec, dp: float, *, fixed=None,
                 correction: bool = True, cfl: float = 0.6, precision: str = "fp64",
                 _slab=None, _grid=None, _dist=None):
        # other kernel families (Laguerre-Gauss) stream the reference
        # gradients g0 (sphb_tl_geometry evaluates any profile)
        wendland = kernel.code == CODE_WENDLAND
        torch = _lib.torch_cuda()
        self.X0 = np.ascontiguousarray(X0, dtype=float)
        self.n, self.dim = self.X0.shape
        self.material = material
        self.kernel = kernel
        self.cfl = float(cfl)
        self.dp = float(dp)
        self.vol0 = np.full(self.n, self.dp**self.dim)
        self.rho0 = material.rho0
        self.fixed = (np.zeros(self.n, dtype=bool) if fixed is None
                      else np.asarray(fixed, dtype=bool))
        self.t = 0.0
        self.steps = 0
        dev = _lib.device()
        self._dev = dev

        # slab ranks (slab.py) bin their owned+halo set with the GLOBAL grid
        self._slab, self._dist = _slab, _dist
        self.grid = (_grid if _grid is not None
                     else make_grid(self.X0, kernel.kappa * kernel.h, None))   # tlsph.py:140
        self.bins = bin_particles(_lib.to_device(self.X0, torch.float64), self.grid)
        if _slab is not None:
            _slab.attach(self.bins.perm.cpu().numpy())
        self.nbr, self.cnt, self.width = ell_from_bins(self.bins, kernel.h, kernel.kappa)
        self.perm = self.bins.perm.long()
        self.rank = self.bins.rank()
        self._nlist = None
        n, d = self.n, self.dim

        vol_s = torch.full((n,), self.dp**d, dtype=torch.float64, device=dev)
        if correction:
            m = torch.empty((n, d, d), dtype=torch.float64, device=dev)
            k = _lib.kernel_struct(kernel)
            _lib.call("sphb_ell_moments", ctypes.byref(self.grid), n,
                      self.bins.ws.contiguous().data_ptr(), self.nbr.data_ptr(),
                      self.cnt.data_ptr(), vol_s.data_ptr(), ctypes.byref(k), m.data_ptr(),
                      _lib.stream_ptr())
            from .correction import correction_from_moments_device

            b0, _, reg = correction_from_moments_device(m)
            self.n_regularized = int(reg.sum().item())
        else:
            b0 = torch.eye(d, dtype=torch.float64, device=dev).expand(n, d, d).contiguous()
            self.n_regularized = 0
        # engine storage order (neighbors.engine_order) on one GPU
        self.order = self.bins
        if os.environ.get("SPHB_ENGINE_ORDER", "lattice") != "cell":
            self.order, self.nbr, self.cnt = engine_order(self.bins, self.nbr, self.cnt,
                                                          self.width, spacing=self.dp)
            b0 = b0[self.order.q].contiguous()
            self.perm = self.order.perm.long()
            self.rank = self.order.rank()
            if _slab is not None:   # owned / halo slices in the new order
                _slab.attach(self.order.perm.cpu().numpy())
        self._B0_sorted = b0
        fixed_s = _lib.to_device(self.fixed.astype(np.float64), torch.float64)[self.perm]
        self.X0rec = _vec_rec(self.order.ws.t(), n, d, dev)
        self.X0rec[:, 3] = fixed_s
        self.B0rec = _b0_rec(b0, n, d, dev)
        eye = torch.eye(d, dtype=torch.float64, device=dev).expand(n, d, d)
        self.Frec = _f_rec(eye, n, d, dev)
        # Q: three column planes in 3D (tl_common.cuh store_q), one stride for
        # all slab ranks so the fused halo push can address peer planes
        self._q_stride = n
        if d == 3:
            if _slab is not None and _slab.world > 1:
                qs = torch.tensor([n], dtype=torch.float64, device=dev)
                _dist.all_reduce(qs, op=_dist.ReduceOp.MAX)
                self._q_stride = int(qs.item())
            self.Qrec = torch.zeros((3, self._q_stride, 4), dtype=torch.float64, device=dev)
            self._q_halo = [self.Qrec[r] for r in range(3)]
        else:
            self.Qrec = torch.zeros((n, 4), dtype=torch.float64, device=dev)
            self._q_halo = [self.Qrec]
        xs = _lib.to_device(self.X0, torch.float64)[self.perm]
        self.XC = _vec_rec(xs, n, d, dev)
        self.V = torch.zeros((n, 4), dtype=torch.float64, device=dev)
        self.A = torch.zeros_like(self.V)
        self.A[:, 3] = fixed_s            # clamp flag rides in A.w (tl_engine.cu)
        self.Vh = torch.zeros_like(self.V)
        self.scalars = torch.zeros(4, dtype=torch.float64, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)

        lam, g = material.lame
        p = self.params = _lib.TLParams()
        p.dim, p.width, p.n = d, self.width, n
        p.row0, p.nrows = ((_slab.rows.start, _slab.rows.stop - _slab.rows.start)
                           if _slab is not None else (0, n))
        p.h, p.alpha, p.kappa = kernel.h, kernel.alpha, kernel.kappa
        p.vol0, p.rho0, p.lam, p.g = self.dp**d, self.rho0, lam, g
        p.q_stride = self._q_stride
        p.law = LAWS[getattr(material, "law", SVK)]
        self._cfl_h = self.cfl * kernel.h
        self._c_s = material.sound_speed
        # reference gradients g0: recomputed per pair from X0 by default (with
        # engine order + staged pass lists that beats streaming 24 B/pair:
        # C4 0.85 vs 0.96 ms/step); SPHB_TL_GEO=1 streams them when they fit
        # in a quarter of the free memory
        self.g0 = None
        g0_bytes = d * self.width * n * 8
        if not wendland and g0_bytes >= 0.5 * torch.cuda.mem_get_info()[0]:
            raise NotImplementedError("non-Wendland TL kernels stream g0, which does not fit")
        if n and self.width and (not wendland or (
                os.environ.get("SPHB_TL_GEO", "0") != "0"
                and g0_bytes < 0.25 * torch.cuda.mem_get_info()[0])):
            self.g0 = torch.empty(g0_bytes // 8, dtype=torch.float64, device=dev)
            k = _lib.kernel_struct(kernel)
            _lib.call("sphb_tl_geometry", ctypes.byref(self.grid), n,
                      self.order.ws.contiguous().data_ptr(), self.nbr.data_ptr(),
                      self.cnt.data_ptr(), self.width, ctypes.byref(k), self.dp**d,
                      self.g0.data_ptr(), _lib.stream_ptr())
        self._g0_ptr = None if self.g0 is None else self.g0.data_ptr()
        self.lattice = None
        if (_slab is None and self.g0 is None and self.order is not self.bins
                and os.environ.get("SPHB_TL_LATTICE", "1") != "0"):
            self._setup_lattice()
        # optional FP32 mode (north star): FP32 companions of the gathered
        # records (v_half, Q) on the lattice passes; FP64 arithmetic and state
        if precision not in ("fp64", "fp32"):
            raise ValueError("precision must be 'fp64' or 'fp32'")
        self.precision = precision
        if precision == "fp32":
            if self.lattice is None:
                raise NotImplementedError("the TL FP32 mode runs on the lattice passes "
                                          "(a lattice reference configuration, one GPU)")
            self.Vh32 = torch.zeros((n, 4), dtype=torch.float32, device=dev)
            self.Q32 = torch.zeros((3 if d == 3 else 1, self._q_stride, 4),
                                   dtype=torch.float32, device=dev)
            p.vh32, p.q32 = self.Vh32.data_ptr(), self.Q32.data_ptr()
        self._setup_push(dev)
        self._acc_valid = False
        self._host = {}
        self._v_out = False

    # -- host views -----------------------------------------------------------
    def _orig(self, t):
        return t[self.rank].cpu().numpy()

    def _cached(self, name, fn):
        if name not in self._host:
            self._host[name] = fn()
        return self._host[name]

    @property
    def x(self):
        return self._cached("x", lambda: self._orig(self.XC[:, :self.dim]))

    @property
    def v(self):
        """Velocities (caller order).  The array handed out is authoritative
        until the next step: in-place edits (e.g. `system.v[clamp] = 0`,
        cases.py:455) are uploaded before stepping."""
        self._v_out = True
        return self._cached("v", lambda: self._orig(self.V[:, :self.dim]))

    @v.setter
    def v(self, value):
        torch = _lib.torch_cuda()
        vs = _lib.to_device(np.asarray(value, dtype=float).reshape(self.n, self.dim),
                            torch.float64)[self.perm]
        self.V[:, :self.dim] = vs
        self._host.pop("v", None)
        self._v_out = False

    def _sync_in(self):
        if self._v_out and "v" in self._host:
            host_v = self._host.pop("v")
            self.v = host_v
        self._v_out = False

    @property
    def F(self):
        return self._cached("F", lambda: self._orig(_f_unrec(self.Frec, self.n, self.dim)))

    @property
    def B0(self):
        return self._cached("B0", lambda: self._orig(self._B0_sorted))

    @property
    def nlist0(self) -> NeighborList:
        if self._nlist is None:
            starts, idx, r, e = csr_from_bins(self.bins)
            self._nlist = NeighborList(starts, idx, r, e, cutoff=self.grid.cutoff, bins=self.bins)
        return self._nlist

    # -- force evaluation -------------------------------------------------------
    def first_pk(self):
        s = pk2_stress(self.F, self.material)
        return np.einsum("nab,nbc->nac", self.F, s), s

    def _setup_lattice(self):
        """Lattice fast path (csrc/tl_lattice.cu) when the reference
        configuration is a complete box lattice in engine order: the interior
        rows (full stencil) run the lattice passes, the shell rows the
        general ones through a row list.  Needs sphb_tl_lattice_check to
        prove every interior row: its pass-list set and, for the default
        table geometry (per-slot dx and g0, antisymmetric), every pair's
        exact displacement within 1e-12 dp of its slot's; for the exact mode
        (SPHB_TL_TABLE=0, or when the table check fails) bitwise separable
        displacements and r2 near the slot's expansion point."""
        torch = _lib.torch_cuda()
        d, n, dp = self.dim, self.n, self.dp
        if d not in (2, 3) or n == 0 or int(self.grid.slow_axis) != d - 1 or n >= 2**31:
            return
        w = self.X0rec[:, :d]
        lo, hi = w.min(dim=0).values.cpu().numpy(), w.max(dim=0).values.cpu().numpy()
        ext = [int(round((hi[a] - lo[a]) / dp)) + 1 for a in range(d)]
        if int(np.prod(ext)) != n:
            return
        r2 = int(math.floor((self.grid.cutoff / dp) ** 2 * (1.0 + 1e-12)))
        lib = _lib.lib()
        width = int(lib.sphb_tl_lattice_width(d, r2))
        R = math.isqrt(r2)
        if width == 0 or width != self.width or min(ext) <= 2 * R:
            return
        offs = [(x, y, z) for z in (range(-R, R + 1) if d > 2 else [0])
                for y in range(-R, R + 1) for x in range(-R, R + 1)
                if 0 < x * x + y * y + z * z <= r2]
        L = _lib.TLLattice()
        L.width, L.r2 = width, r2
        for a in range(3):
            L.n[a] = ext[a] if a < d else 1
        L.n_interior = int(np.prod([e - 2 * R for e in ext]))
        stride = [1, ext[0], ext[0] * (ext[1] if d > 1 else 1)]
        rep = [e // 2 for e in ext] + [0] * (3 - d)
        irep = sum(rep[a] * stride[a] for a in range(3))
        rows = [irep] + [irep + sum(o[a] * stride[a] for a in range(3)) for o in offs]
        xw = self.X0rec[torch.tensor(rows, device=self._dev), :d].cpu().numpy()
        h = self.kernel.h
        c5v = -5.0 * (self.kernel.alpha / h * dp**d) / h      # tl_engine.cu ref_gradient
        dxk = xw[0] - xw[1:]                          # (width, d), representative row
        # table geometry: antisymmetric (slot W-1-k is the mirror of slot k
        # in the canonical order), so sum_k g[k] = 0 exactly
        half = width // 2
        dxt = dxk.copy()
        dxt[:half] = -dxk[::-1][:half]
        for k in range(width):
            dx = dxk[k]
            r2k = float(np.sum(dx * dx))
            r = math.sqrt(r2k)
            t = 1.0 - 0.5 * r / h
            L.r2k[k] = r2k
            L.f[k] = c5v * ((t * t) * t)
            L.df[k] = 3.0 * c5v * t * t * (-0.25 / (h * r))
            rt = math.sqrt(float(np.sum(dxt[k] * dxt[k])))
            tt = 1.0 - 0.5 * rt / h
            ft = c5v * ((tt * tt) * tt)
            for a in range(d):
                L.dx[k][a] = float(dxt[k][a])
                L.g[k][a] = ft * float(dxt[k][a])
        idx = torch.arange(n, device=self._dev)
        coord = [idx % ext[0], (idx // ext[0]) % ext[1] if d > 1 else None,
                 idx // (ext[0] * ext[1]) if d > 2 else None]
        inner = torch.ones(n, dtype=torch.bool, device=self._dev)
        for a in range(d):
            inner &= (coord[a] >= R) & (coord[a] < ext[a] - R)
        self._shell = torch.nonzero(~inner).flatten().to(torch.int32).contiguous()
        L.shell, L.n_shell = self._shell.data_ptr(), int(self._shell.numel())
        # compact shell pass list, column-major over the shell rows (coalesced
        # reads; the full list's shell rows are scattered over its columns)
        sh = self._shell.long()
        self._shell_nbr = self.nbr.view(-1, n)[:, sh].contiguous()
        self._shell_cnt = self.cnt[sh].contiguous()
        L.shell_nbr, L.shell_cnt = self._shell_nbr.data_ptr(), self._shell_cnt.data_ptr()
        # table geometry (default; SPHB_TL_TABLE=0 keeps the exact separable
        # geometry): every interior pair within 1e-12 dp of its slot's dx,
        # else the exact mode's proof (bitwise separability, r2 near r2k)
        modes = [(1, 1e-12 * dp), (0, 1e-10)]
        if os.environ.get("SPHB_TL_TABLE", "1") == "0":
            modes = modes[1:]
        for table, tol in modes:
            L.table = table
            bad = torch.zeros(1, dtype=torch.int64, device=self._dev)
            _lib.call("sphb_tl_lattice_check", ctypes.byref(self.params), ctypes.byref(L),
                      self.X0rec.data_ptr(), self.nbr.data_ptr(), self.cnt.data_ptr(), tol,
                      bad.data_ptr(), _lib.stream_ptr())
            if int(bad.item()) == 0:
                self.lattice = L
                # table mode: dense 3D Q records (no X0 padding, 24-byte column
                # gathers in pass B); every Q writer and reader honours the flag
                self.params.q_dense = int(table == 1 and d == 3 and self._q_stride == n)
                if table == 1 and d == 3:
                    self._setup_uniform_b0(L, R, ext)
                return

    def _setup_uniform_b0(self, L, R, ext):
        """Uniform B0 on the interior rows (table mode, 3D): every interior
        row has the full canonical stencil, so its correction matrix B0
        (tlsph.py:140-141) is the same matrix up to rounding; when every
        interior record equals b0 (the first interior row's) to 1e-12 of
        max|b0| (sphb_tl_uniform_b0_check), pass A takes B0 from b0 there
        and reads no B0 records (48 of its streamed bytes per row).  The
        shell rows keep their own records."""
        if os.environ.get("SPHB_TL_UNIFORM_B0", "1") == "0":
            return
        torch = _lib.torch_cuda()
        n = self.n
        i0 = R + ext[0] * (R + ext[1] * R)
        b0 = torch.cat([self.B0rec[:4 * n].view(n, 4)[i0],
                        self.B0rec[4 * n:].view(n, 2)[i0]]).contiguous()
        bad = torch.zeros(1, dtype=torch.int64, device=self._dev)
        _lib.call("sphb_tl_uniform_b0_check", ctypes.byref(self.params), ctypes.byref(L),
                  self.B0rec.data_ptr(), b0.data_ptr(), 1e-12, bad.data_ptr(),
                  _lib.stream_ptr())
        if int(bad.item()) == 0:
            L.uniform_b0 = 1
            for e, v in enumerate(b0.cpu().tolist()):
                L.b0[e] = v

    def _pass_b(self, update_v):
        st = _lib.stream_ptr()
        if self.lattice is not None:
            _lib.call("sphb_tl_pass_b_lattice", ctypes.byref(self.params),
                      ctypes.byref(self.lattice), self.X0rec.data_ptr(), self.nbr.data_ptr(),
                      self.cnt.data_ptr(), self.Qrec.data_ptr(), self.Vh.data_ptr(),
                      self.A.data_ptr(), self.V.data_ptr(), self.scalars.data_ptr(), update_v,
                      self.err.data_ptr(), st)
            return
        _lib.call("sphb_tl_pass_b", ctypes.byref(self.params), self.X0rec.data_ptr(),
                  self.nbr.data_ptr(), self.cnt.data_ptr(), self._g0_ptr, self.Qrec.data_ptr(),
                  self.Vh.data_ptr(), self.A.data_ptr(), self.V.data_ptr(),
                  self.scalars.data_ptr(), update_v, self.err.data_ptr(), st)

    def _accelerations_dev(self):
        st = _lib.stream_ptr()
        _lib.call("sphb_tl_stress", ctypes.byref(self.params), self.Frec.data_ptr(),
                  self.B0rec.data_ptr(), self.X0rec.data_ptr(), self.Qrec.data_ptr(), st)
        self._halo(*self._q_halo)
        self._pass_b(0)
        self._halo(self.A)
        self._acc_valid = True

    def _halo(self, *bufs):
        if self._slab is not None:
            self._slab.exchange(self._dist, list(bufs), reuse=True)

    def _setup_push(self, dev):
        """Fused halo push (SPHB_HALO_PUSH=1): pass A stores the boundary
        layers' Q records and pass B their A / V records straight into the
        neighbour ranks' halo rows (peer memory)."""
        self._push = None
        if not (self._slab is not None and self._slab.world > 1
                and os.environ.get("SPHB_HALO_PUSH", "0") == "1"):
            return
        torch = _lib.torch_cuda()
        self._push = self._slab.share_buffers(self._dist, [self.Qrec, self.A, self.V])
        self._push_token = torch.zeros(1, dtype=torch.int32, device=dev)

    def _set_push(self, on: bool):
        p = self.params
        p.push_q_prev = p.push_q_next = p.push_a_prev = p.push_a_next = None
        p.push_v_prev = p.push_v_next = None
        if not on or self._push is None:
            return
        sl = self._slab
        if "prev" in self._push:
            (q, a, v), at = self._push["prev"]
            p.push_q_prev, p.push_a_prev, p.push_v_prev = q, a, v
            p.push_lo0, p.push_lo1, p.push_prev_at = sl.send_lo.start, sl.send_lo.stop, at
        if "next" in self._push:
            (q, a, v), at = self._push["next"]
            p.push_q_next, p.push_a_next, p.push_v_next = q, a, v
            p.push_hi0, p.push_hi1, p.push_next_at = sl.send_hi.start, sl.send_hi.stop, at

    def _reduce_speed(self):
        if self._slab is not None and self._slab.world > 1:
            self._dist.all_reduce(self.scalars[2:3], op=self._dist.ReduceOp.MAX)

    def owned(self):
        """(global ids, x, v, F) of the rows this system updates (slab ranks)."""
        rows = self._slab.rows if self._slab is not None else slice(0, self.n)
        ids = self.perm[rows].cpu().numpy()
        if self._slab is not None:
            ids = self._slab.local_ids[ids]
        x = self.XC[rows, :self.dim].cpu().numpy()
        v = self.V[rows, :self.dim].cpu().numpy()
        F = _f_unrec(self.Frec, self.n, self.dim, rows).cpu().numpy()
        return ids, x, v, F

    def accelerations(self):
        """Corrected TL momentum rate / rho0 (tlsph.py:164-171), caller order."""
        self._accelerations_dev()
        return self._orig(self.A[:, :self.dim])

    def deformation_rates(self):
        """dF_i = [sum_j V0 (v_j - v_i) (x) grad0 W_ij] B0_i (tlsph.py:173-176),
        via the reference-order CSR operator (sphb_tl_deformation_rates_csr)."""
        torch = _lib.torch_cuda()
        from .correction import pair_gradients_device

        nl = self.nlist0
        starts, idx, _, _ = nl.device_csr()
        g0 = (pair_gradients_device(nl, self.kernel, None) * (self.dp**self.dim)).contiguous()
        v = _lib.to_device(self.v, torch.float64)
        b0 = _lib.to_device(self.B0, torch.float64)
        dF = torch.empty((self.n, self.dim, self.dim), dtype=torch.float64, device=self._dev)
        _lib.call("sphb_tl_deformation_rates_csr", self.n, self.dim, starts.data_ptr(),
                  idx.data_ptr(), g0.data_ptr(), v.data_ptr(), b0.data_ptr(), dF.data_ptr(),
                  _lib.stream_ptr())
        return dF.cpu().numpy()

    def _speed_max(self):
        _lib.call("sphb_tl_speed_max", ctypes.byref(self.params), self.V.data_ptr(),
                  self.scalars.data_ptr(), _lib.stream_ptr())
        self._reduce_speed()

    def stable_dt(self) -> float:
        """cfl h / (c_s + max|v|) (tlsph.py:178-180)."""
        self._sync_in()
        self._speed_max()
        vmax = float(self.scalars[2].item())
        return self._cfl_h / (self._c_s + vmax)

    def _one_step(self, dt_override: float):
        st = _lib.stream_ptr()
        self._set_push(True)
        _lib.call("sphb_set_dt", self._cfl_h, self._c_s, dt_override, self.scalars.data_ptr(),
                  self.err.data_ptr(), st)
        if self.lattice is not None:
            # kick, then pass A over the interior (lattice) and shell rows
            _lib.call("sphb_tl_kick", ctypes.byref(self.params), self.V.data_ptr(),
                      self.A.data_ptr(), self.Vh.data_ptr(), self.scalars.data_ptr(), st)
            _lib.call("sphb_tl_pass_a_lattice", ctypes.byref(self.params),
                      ctypes.byref(self.lattice), self.X0rec.data_ptr(), self.B0rec.data_ptr(),
                      self.nbr.data_ptr(), self.cnt.data_ptr(), self.Vh.data_ptr(),
                      self.XC.data_ptr(), self.Frec.data_ptr(), self.Qrec.data_ptr(),
                      self.scalars.data_ptr(), self.err.data_ptr(), st)
        else:
            _lib.call("sphb_tl_pass_a", ctypes.byref(self.params), self.X0rec.data_ptr(),
                      self.B0rec.data_ptr(), self.nbr.data_ptr(), self.cnt.data_ptr(),
                      self._g0_ptr, self.V.data_ptr(), self.A.data_ptr(), self.Vh.data_ptr(),
                      self.XC.data_ptr(), self.Frec.data_ptr(), self.Qrec.data_ptr(),
                      self.scalars.data_ptr(), self.err.data_ptr(), st)
        if self._push is not None:                  # Q halos were pushed by pass A
            self._dist.all_reduce(self._push_token)
        else:
            self._halo(*self._q_halo)
        self._pass_b(1)
        self._set_push(False)
        if self._push is None:                      # else pushed; the max orders them
            self._halo(self.V, self.A)
        self._reduce_speed()

    def _raise_if_bad(self):
        if self._slab is not None and self._slab.world > 1:
            e = self.err.clone()
            self._dist.all_reduce(e, op=self._dist.ReduceOp.MAX)
            err = int(e.item())
        else:
            err = int(self.err.item())
        if err:
            self.err.zero_()
            raise SolidStateError(f"deformation gradient inverted (flags {err}) "
                                  f"at step {self.steps}")

    def step(self, dt: float | None = None) -> float:
        """Kick-drift-kick update of (v, x, F) (tlsph.py:182-206)."""
        self._sync_in()
        if dt is None:
            dt = self.stable_dt()
        if not self._acc_valid:
            self._accelerations_dev()
        self._one_step(float(dt))
        self._host.clear()
        self._raise_if_bad()
        self.t += dt
        self.steps += 1
        return dt

    def advance(self, n_steps: int, dt: float | None = None, *, graph: bool | None = None) -> None:
        """n_steps steps without host synchronisation; the error word is read
        once at the end (SolidStateError).  With `graph` (default when
        n_steps >= 8) one step is captured as a CUDA graph and replayed."""
        if n_steps <= 0:
            return
        self._sync_in()
        if not self._acc_valid:
            self._accelerations_dev()
        dto = 0.0 if dt is None else float(dt)
        if dt is None:
            self._speed_max()
        self.scalars[1] = 0.0
        if graph is None:
            graph = n_steps >= 8 and self._slab is None
        if graph:
            g, per = self._step_graph(dto)
            for _ in range(n_steps // per):
                g.replay()
            for _ in range(n_steps % per):
                self._one_step(dto)
        else:
            for _ in range(n_steps):
                self._one_step(dto)
        self._host.clear()
        self._raise_if_bad()
        self.t += float(self.scalars[1].item())
        self.steps += n_steps

    def _step_graph(self, dt_override: float):
        torch = _lib.torch_cuda()
        if getattr(self, "_graphs", None) is None:
            self._graphs = {}
        from .eulerian import graph_steps

        per = graph_steps()          # steps per replay (amortises replay latency)
        g = self._graphs.get(dt_override)
        if g is None:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(per):
                    self._one_step(dt_override)
            torch.cuda.synchronize()
            self._graphs[dt_override] = g
        return g, per

    # -- diagnostics ------------------------------------------------------------
    def von_mises_field(self):
        """Per-particle von Mises stress (tlsph.py:210-212)."""
        _, s = self.first_pk()
        return von_mises(self.F, s)

    def energies(self):
        """(kinetic, strain) energy; strain energy 1/2 S:E for SVK, the
        stored energy G/2 (tr C - d) - G ln J + lam/2 (ln J)^2 for
        Neo-Hookean."""
        eye = np.eye(self.dim)
        C = np.einsum("nba,nbc->nac", self.F, self.F)
        if getattr(self.material, "law", SVK) == NEO_HOOKEAN:
            lam, g = self.material.lame
            ln_j = 0.5 * np.log(np.linalg.det(C))
            w = 0.5 * g * (np.trace(C, axis1=1, axis2=2) - self.dim) - g * ln_j \
                + 0.5 * lam * ln_j**2
            e_strain = float(np.sum(self.vol0 * w))
        else:
            _, s = self.first_pk()
            strain = 0.5 * (C - eye)
            e_strain = 0.5 * float(np.sum(self.vol0 * np.einsum("nab,nab->n", s, strain)))
        e_kin = 0.5 * float(np.sum(self.rho0 * self.vol0 * np.sum(self.v**2, axis=1)))
        return e_kin, e_strain

    def momentum(self):
        return (self.rho0 * self.vol0[:, None] * self.v).sum(axis=0)
