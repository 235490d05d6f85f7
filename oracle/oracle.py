"""CPU ORACLE — test infrastructure only, never the product path.

Python side of the oracle: numpy glue around the plain-C loops in
sph_oracle.c, restating the reference package (pkg/src/sph_trunc of arXiv
2405.05155) function by function.  Used by tests/ (as the checker of the CUDA
path), by __graft_entry__.smoke(), and by bench.py's cpu_baseline and
`--impl reference` legs (as the timed CPU baseline, "kind": "port").

Pinned against the reference by tests/test_oracle_golden.py: golden vectors
written by tests/golden/make_golden.py from the reference itself, plus every
known value of the reference's own unit tests.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

_P = C.c_void_p
_I = C.c_int64
_D = C.c_double

_SIGS = {
    "orc_bin": (_P, [_P, _I, _I, _P, _P, _P, _P, _I, _D]),
    "orc_bin_free": (None, [_P]),
    "orc_count": (None, [_P, _P]),
    "orc_fill": (None, [_P, _P, _P, _P, _P]),
    "orc_unity_sums": (None, [_I, _P, _P, _P, _P, _I, _D, _D, _D, _P]),
    "orc_pressure_accel": (None, [_I, _I, _P, _P, _P, _P, _P, _I, _D, _D, _D, _D, _D, _P]),
    "orc_moment_matrices": (None, [_I, _I, _P, _P, _P, _P, _P, _I, _D, _D, _D, _P]),
    "orc_pair_gradients": (None, [_I, _I, _P, _P, _P, _P, _I, _D, _D, _D, _P, _P]),
    "orc_rhs_wc": (None, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _D, _D, _P, _P, _P, _P]),
    "orc_rhs_hllc": (None, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "orc_tl_accelerations": (None, [_I, _I, _P, _P, _P, _P, _D, _P]),
    "orc_tl_deformation_rates": (None, [_I, _I, _P, _P, _P, _P, _P, _P]),
    "orc_weak_gradient": (None, [_I, _I, _P, _P, _P, _P, _P, _P]),
    "orc_max_threads": (C.c_int, []),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def threads() -> int:
    return int(lib().orc_max_threads())


# ------------------------------------------------------------ neighbours
@dataclass
class NeighborList:
    starts: np.ndarray
    idx: np.ndarray
    r: np.ndarray
    e: np.ndarray
    cutoff: float

    @property
    def n(self):
        return self.starts.shape[0] - 1

    @property
    def counts(self):
        return np.diff(self.starts)


def build_neighbors(positions, cutoff, box=None) -> NeighborList:
    """neighbors.py:171-210 (grid set-up in numpy, loops in C)."""
    pos = np.ascontiguousarray(np.asarray(positions, dtype=float))
    n, d = pos.shape
    if box is not None:
        box_arr = np.asarray(box, dtype=float)
        wrapped = pos % box_arr
        extent = box_arr
    else:
        box_arr = np.ones(d)
        lo = pos.min(axis=0)
        wrapped = pos - lo
        extent = np.maximum(wrapped.max(axis=0), cutoff)
    ncell = np.maximum((extent / cutoff).astype(np.int64), 1)
    inv_cell = ncell / box_arr if box is not None else np.full(d, 1.0 / cutoff)
    strides = np.ones(d, dtype=np.int64)
    for a in range(1, d):
        strides[a] = strides[a - 1] * ncell[a - 1]
    wrapped = np.ascontiguousarray(wrapped)
    inv_cell = np.ascontiguousarray(inv_cell, dtype=float)
    box_c = np.ascontiguousarray(box_arr, dtype=float)
    L = lib()
    h = L.orc_bin(_p(wrapped), n, d, _p(inv_cell), _p(ncell), _p(strides), _p(box_c),
                  int(box is not None), float(cutoff))
    try:
        starts = np.zeros(n + 1, dtype=np.int64)
        L.orc_count(h, _p(starts))
        m = int(starts[-1])
        idx = np.empty(m, dtype=np.int32)
        r = np.empty(m)
        e = np.empty((m, d))
        L.orc_fill(h, _p(starts), _p(idx), _p(r), _p(e))
    finally:
        L.orc_bin_free(h)
    return NeighborList(starts, idx, r, e, float(cutoff))


def pair_set(nl) -> np.ndarray:
    """Sorted (i, j) int64 pairs of a CSR list (canonical form for set equality)."""
    rows = np.repeat(np.arange(nl.n, dtype=np.int64), np.diff(nl.starts))
    key = rows * (nl.n + 1) + nl.idx.astype(np.int64)
    return np.sort(key)


# ------------------------------------------------------------ operators
def sph_unity_sum(nl, vols, spec):
    out = np.empty(nl.n)
    v = np.ascontiguousarray(vols, dtype=float)
    lib().orc_unity_sums(nl.n, _p(nl.starts), _p(nl.idx), _p(nl.r), _p(v), spec.code, spec.h,
                         spec.alpha, spec.kappa, _p(out))
    return out


def relax_accelerations(nl, vols, spec, p0=1.0, rho0=1.0):
    d = nl.e.shape[1]
    acc = np.empty((nl.n, d))
    v = np.ascontiguousarray(vols, dtype=float)
    lib().orc_pressure_accel(nl.n, d, _p(nl.starts), _p(nl.idx), _p(nl.r), _p(nl.e), _p(v),
                             spec.code, spec.h, spec.alpha, spec.kappa, p0, rho0, _p(acc))
    return acc


def moment_matrices(nl, vols, spec):
    d = nl.e.shape[1]
    m = np.empty((nl.n, d, d))
    v = np.ascontiguousarray(vols, dtype=float)
    lib().orc_moment_matrices(nl.n, d, _p(nl.starts), _p(nl.idx), _p(nl.r), _p(nl.e), _p(v),
                              spec.code, spec.h, spec.alpha, spec.kappa, _p(m))
    return m


def _row_chunks(n, fn, parts=None):
    """Run fn(slice) over contiguous row chunks on host threads (numpy's
    gufuncs and elementwise loops release the GIL); every row is computed by
    the same numpy call as unchunked, so results are bit-identical."""
    from concurrent.futures import ThreadPoolExecutor

    parts = parts or max(1, min(threads(), 64))
    if n < 8192 or parts == 1:
        return [fn(slice(0, n))]
    edges = np.linspace(0, n, parts + 1).astype(np.int64)
    with ThreadPoolExecutor(parts) as ex:
        return list(ex.map(lambda k: fn(slice(int(edges[k]), int(edges[k + 1]))), range(parts)))


def correction_matrices(nl, vols, spec):
    """correction.py:64-81 with numpy's LAPACK, as the reference does.
    Returns (B, det(-M), n_regularized)."""
    m = moment_matrices(nl, vols, spec)
    parts = _row_chunks(m.shape[0], lambda sl: _correction_rows(m[sl]))
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]),
            int(sum(p[2] for p in parts)))


def _correction_rows(m):
    n, d, _ = m.shape
    u, s, vt = np.linalg.svd(m)
    floor = 1e-4 * np.maximum(s[:, :1], 1e-300)
    clamped = np.any(s < floor, axis=1)
    s_reg = np.maximum(s, floor)
    minv = np.einsum("nba,nb,ncb->nac", vt, 1.0 / s_reg, u)
    det_neg = np.linalg.det(-m)
    theta = np.clip(det_neg / 1e-6, 0.0, 1.0)
    b = theta[:, None, None] * (-minv) + (1.0 - theta)[:, None, None] * np.eye(d)
    return b, det_neg, int((clamped | (theta < 1.0)).sum())


def pair_gradients(nl, spec, b=None):
    d = nl.e.shape[1]
    gw = np.empty((nl.idx.shape[0], d))
    bb = None if b is None else np.ascontiguousarray(b, dtype=float)
    lib().orc_pair_gradients(nl.n, d, _p(nl.starts), _p(nl.idx), _p(nl.r), _p(nl.e),
                             spec.code, spec.h, spec.alpha, spec.kappa, _p(bb), _p(gw))
    return gw


def weak_gradient(nl, f, vols, spec, b=None):
    """approx.py:74-86."""
    d = nl.e.shape[1]
    gw = np.ascontiguousarray(pair_gradients(nl, spec, b))
    out = np.empty((nl.n, d))
    lib().orc_weak_gradient(nl.n, d, _p(nl.starts), _p(nl.idx),
                            _p(np.ascontiguousarray(f, dtype=float)),
                            _p(np.ascontiguousarray(vols, dtype=float)), _p(gw), _p(out))
    return out


def _profile_deriv(code, q):
    if code == 0:
        t = 1.0 - 0.5 * q
        return -5.0 * q * t**3
    return q * (-3.0 + (5.0 / 3.0) * q**2 - q**4 / 3.0) * np.exp(-(q**2))


# ------------------------------------------------------------ relaxation
def relax_steps(pos, spec, box, dp, n_updates, p0=1.0, rho0=1.0, step_scale=0.2):
    """relaxation.py:157-195 loop body with no stop tests."""
    pos = np.array(pos, dtype=float)
    n, d = pos.shape
    vols = np.full(n, dp**d)
    cutoff = spec.kappa * spec.h
    dt2 = step_scale * spec.h**2 * rho0 / p0
    cap = 0.25 * dp
    box = np.asarray(box, dtype=float)
    residuals = []
    for step in range(n_updates + 1):
        nl = build_neighbors(pos, cutoff, box)
        acc = relax_accelerations(nl, vols, spec, p0, rho0)
        residuals.append(float(np.mean(np.linalg.norm(acc, axis=1)) * spec.h * rho0 / p0))
        if step == n_updates:
            break
        dx = acc * dt2
        norms = np.linalg.norm(dx, axis=1)
        over = norms > cap
        if np.any(over):
            dx[over] *= (cap / norms[over])[:, None]
        pos += dx
        pos %= box
    return pos, np.asarray(residuals)


# ------------------------------------------------ shape-bounded relaxation
class Shape:
    """Signed-distance shapes of geometry.py:16-126 (kind: "circle",
    "rectangle", "semicircle")."""

    def __init__(self, kind, center=None, radius=None, lo=None, hi=None, normal=None):
        self.kind = kind
        self.center = None if center is None else np.asarray(center, dtype=float)
        self.radius = radius
        self.lo = None if lo is None else np.asarray(lo, dtype=float)
        self.hi = None if hi is None else np.asarray(hi, dtype=float)
        self.normal = None if normal is None else np.asarray(normal, dtype=float)

    def bounds(self):
        if self.kind == "rectangle":
            return self.lo, self.hi
        return self.center - self.radius, self.center + self.radius

    def signed_distance(self, x):
        x = np.asarray(x, dtype=float)
        if self.kind == "circle":                                # geometry.py:37-39
            return np.linalg.norm(x - self.center, axis=-1) - self.radius
        if self.kind == "rectangle":                             # geometry.py:60-69
            q = np.abs(x - 0.5 * (self.lo + self.hi)) - 0.5 * (self.hi - self.lo)
            return (np.linalg.norm(np.maximum(q, 0.0), axis=-1)
                    + np.minimum(np.max(q, axis=-1), 0.0))
        p = x - self.center                                      # geometry.py:107-126
        a = p @ self.normal
        tnorm = np.linalg.norm(p - np.multiply.outer(a, self.normal), axis=-1)
        d_in = np.maximum(np.linalg.norm(p, axis=-1) - self.radius, a)
        tc = np.minimum(tnorm, self.radius)
        d_out = np.sqrt(np.maximum(tnorm - tc, 0.0) ** 2 + a**2)
        return np.where(a <= 0.0, d_in, d_out)

    def gradient(self, x, eps=1e-7):
        """geometry.py:137-147."""
        x = np.atleast_2d(np.asarray(x, dtype=float))
        g = np.empty_like(x)
        for a in range(x.shape[1]):
            step = np.zeros(x.shape[1])
            step[a] = eps
            g[:, a] = (self.signed_distance(x + step) - self.signed_distance(x - step)) / (2 * eps)
        nrm = np.linalg.norm(g, axis=1, keepdims=True)
        nrm[nrm == 0.0] = 1.0
        return g / nrm

    def lattice_fill(self, dp):
        """geometry.py:150-170."""
        lo, hi = self.bounds()
        counts = np.maximum(np.round((hi - lo) / dp).astype(int), 1)
        axes = [lo[a] + (np.arange(counts[a]) + 0.5) * dp for a in range(len(lo))]
        mesh = np.meshgrid(*axes, indexing="ij")
        pts = np.stack([m.ravel() for m in mesh], axis=1)
        return pts[self.signed_distance(pts) < 0.0]


def kernel_value(spec, r):
    """kernels.py:132-146."""
    q = np.asarray(r, dtype=float) / spec.h
    out = np.zeros_like(q)
    inside = q <= spec.kappa
    qi = q[inside]
    if spec.code == 0:
        t = 1.0 - 0.5 * qi
        out[inside] = spec.alpha * t**4 * (2.0 * qi + 1.0)
    else:
        out[inside] = spec.alpha * (1.0 - 0.5 * qi**2 + qi**4 / 6.0) * np.exp(-(qi**2))
    return out


def wall_table(spec, n_s=256, n_t=2000):
    """_wall_kernel_table (relaxation.py:92-111)."""
    cut = spec.kappa * spec.h
    s = np.linspace(0.0, cut, n_s)
    if spec.dim == 1:
        return s, kernel_value(spec, s)
    t = (np.arange(n_t) + 0.5) * (cut / n_t)
    rr = np.sqrt(s[:, None] ** 2 + t[None, :] ** 2)
    if spec.dim == 2:
        return s, 2.0 * np.sum(kernel_value(spec, rr), axis=1) * (cut / n_t)
    return s, 2.0 * np.pi * np.sum(kernel_value(spec, rr) * t[None, :], axis=1) * (cut / n_t)


def wall_confinement(spec, depth):
    s, w2 = wall_table(spec)
    return np.interp(np.asarray(depth, dtype=float), s, w2, right=0.0)


def relax_shape(shape, spec, dp, max_steps, p0=1.0, rho0=1.0, step_scale=0.2):
    """relax() with box=None (relaxation.py:132-210), no stop tests besides
    max_steps; returns (best-residual positions, residuals, best_step)."""
    pos = shape.lattice_fill(dp).copy()
    n, d = pos.shape
    vols = np.full(n, dp**d)
    cutoff = spec.kappa * spec.h
    dt2 = step_scale * spec.h**2 * rho0 / p0
    cap = 0.25 * dp
    surf_tol = 1e-9 * dp
    residuals, best, best_step, best_pos = [], np.inf, 0, pos.copy()
    for step in range(max_steps + 1):
        nl = build_neighbors(pos, cutoff)
        acc = relax_accelerations(nl, vols, spec, p0, rho0)
        depth = -shape.signed_distance(pos)
        near = depth < cutoff
        if np.any(near):
            nrm = shape.gradient(pos[near])
            acc[near] -= (2.0 * p0 / rho0) * wall_confinement(spec, depth[near])[:, None] * nrm
        res = float(np.mean(np.linalg.norm(acc, axis=1)) * spec.h * rho0 / p0)
        residuals.append(res)
        if res < best:
            best, best_step, best_pos = res, step, pos.copy()
        if step == max_steps:
            break
        dx = acc * dt2
        norms = np.linalg.norm(dx, axis=1)
        over = norms > cap
        if np.any(over):
            dx[over] *= (cap / norms[over])[:, None]
        pos += dx
        outside = shape.signed_distance(pos) > surf_tol
        for _ in range(3):                                      # relaxation.py:120-129
            if not np.any(outside):
                break
            sd = shape.signed_distance(pos[outside])
            pos[outside] -= sd[:, None] * shape.gradient(pos[outside])
            outside = shape.signed_distance(pos) > 1e-12
    return best_pos, np.asarray(residuals), best_step


# ------------------------------------------------------------ WC Eulerian
class StateRejected(RuntimeError):
    """SolverError of the reference (eulerian.py:40-41)."""


class EulerianWC:
    """EulerianSolver, WC branch (eulerian.py:473-643): periodic or with a
    ghost frame, optional wall-force tags (:515-519, 605-606)."""

    def __init__(self, pos, vol, rho, mom, spec, c_art, rho0=1.0, mu=0.0, cfl=0.5, box=None,
                 correction=True, ghosts=None, n_int=None, wall_tag=None):
        self.spec, self.c_art, self.rho0, self.mu, self.cfl = spec, c_art, rho0, mu, cfl
        self.nl = build_neighbors(pos, spec.kappa * spec.h, box)
        self.vol = np.asarray(vol, dtype=float)
        self.rho = np.array(rho, dtype=float)
        self.mom = np.array(mom, dtype=float)
        self.n, self.d = self.mom.shape
        self.n_int = self.n if n_int is None else int(n_int)
        self.ghosts = ghosts
        b = correction_matrices(self.nl, self.vol, spec)[0] if correction else None
        if b is not None and ghosts is not None:       # eulerian.py:499-501
            b[self.n_int:] = b[np.asarray(ghosts.src, dtype=np.int64)]
        self.B = b
        gw = pair_gradients(self.nl, spec, b)
        m = self.nl.idx.shape[0]
        self.gwv = np.empty_like(gw)
        self.viscv = np.empty(m)

        def pair_rows(sl):                              # eulerian.py:506-513
            vj = self.vol[self.nl.idx[sl]]
            self.gwv[sl] = gw[sl] * vj[:, None]
            q = self.nl.r[sl] / spec.h
            dw = np.where(q <= spec.kappa,
                          (spec.alpha / spec.h) * _profile_deriv(spec.code, q), 0.0)
            self.viscv[sl] = 2.0 * dw / self.nl.r[sl] * vj

        _row_chunks(m, pair_rows)
        del gw
        self.t = 0.0
        self.wall_tag = None
        if wall_tag is not None:
            self.wall_tag = np.zeros(self.n, dtype=np.int8)
            self.wall_tag[np.asarray(wall_tag, dtype=np.int64)] = 1
        self.wall_force = np.zeros(self.d)
        self.wall_force_series = []

    def apply_boundaries(self):
        """Ghost refresh, WC kinds (eulerian.py:371-433)."""
        g = self.ghosts
        if g is None:
            return
        ni, g0 = self.n_int, self.n_int
        kind = np.asarray(g.kind)
        src = np.asarray(g.src, dtype=np.int64)
        vel = self.mom[:ni] / self.rho[:ni, None]
        rho, mom = self.rho, self.mom
        m = kind == 0
        if np.any(m):
            rho[g0:][m] = rho[src[m]]
            mom[g0:][m] = mom[src[m]]
        m = kind == 1
        if np.any(m):
            s, nrm = src[m], np.asarray(g.normal)[m]
            vs = vel[s]
            vg = vs - 2.0 * np.sum(vs * nrm, axis=1, keepdims=True) * nrm
            rho[g0:][m] = rho[s]
            mom[g0:][m] = rho[s, None] * vg
        m = kind == 2
        if np.any(m):
            s = src[m]
            rho[g0:][m] = rho[s]
            mom[g0:][m] = rho[s, None] * np.asarray(g.wall_v)[m]
        m = kind == 3
        if np.any(m):
            fx = np.asarray(g.fixed)[m]
            rho[g0:][m] = fx[:, 0]
            mom[g0:][m] = fx[:, 1:1 + self.d]
        m = kind == 5
        if np.any(m):
            s, nrm = src[m], np.asarray(g.normal)[m]
            lam = np.asarray(g.blend)[m][:, None]
            vs = vel[s]
            vn = np.sum(vs * nrm, axis=1, keepdims=True) * nrm
            rho[g0:][m] = rho[s]
            mom[g0:][m] = rho[s, None] * (vs - 2.0 * lam * vn)

    def rhs(self):
        p = self.c_art**2 * (self.rho - self.rho0)
        v = np.ascontiguousarray(self.mom / self.rho[:, None])
        drho = np.empty(self.n)
        dmom = np.zeros((self.n, self.d))
        wf = None if self.wall_tag is None else np.empty((self.n_int, self.d))
        lib().orc_rhs_wc(self.n_int, self.d, _p(self.nl.starts), _p(self.nl.idx), _p(self.nl.e),
                         _p(self.gwv), _p(self.viscv), _p(self.rho), _p(v), _p(p), self.c_art,
                         self.mu, _p(drho), _p(dmom), _p(self.wall_tag), _p(wf))
        if wf is not None:
            self.wall_force = wf.sum(axis=0)
        return drho, dmom

    def compute_dt(self):
        ni = self.n_int
        speed = self.c_art + np.linalg.norm(self.mom[:ni] / self.rho[:ni, None], axis=1)
        return self.cfl * self.spec.h / float(speed.max())

    retries = 0

    def _checked_rhs(self):
        """rhs() with the reference's rejections: eos_eval raises on rho <= 0
        (eulerian.py:70-71, 535), a non-finite momentum flux raises
        (:548-550)."""
        if not np.all(self.rho > 0.0):
            raise StateRejected("non-positive density")
        drho, dmom = self.rhs()
        if not np.all(np.isfinite(dmom[:self.n_int])):
            raise StateRejected("NaN flux")
        return drho, dmom

    def _substep(self, dt):
        """eulerian.py:610-643: midpoint substep; on rejection the interior
        is restored to the substep start and t is not advanced."""
        ni = self.n_int
        rho0, mom0 = self.rho[:ni].copy(), self.mom[:ni].copy()
        try:
            self.apply_boundaries()
            drho, dmom = self._checked_rhs()
            self.rho[:ni] = rho0 + 0.5 * dt * drho[:ni]
            self.mom[:ni] = mom0 + 0.5 * dt * dmom[:ni]
            self.apply_boundaries()
            drho, dmom = self._checked_rhs()
            self.rho[:ni] = rho0 + dt * drho[:ni]
            self.mom[:ni] = mom0 + dt * dmom[:ni]
            if not np.all(self.rho[:ni] > 0.0):
                raise StateRejected("non-positive density after step")
        except StateRejected:
            self.rho[:ni], self.mom[:ni] = rho0, mom0
            raise
        self.t += dt

    def _fields(self):
        return [self.rho, self.mom]

    def step(self, dt=None):
        """eulerian.py:562-608: one step with retry-with-halving.  A failed
        substep restarts the whole step from its start state at dt/2^k; t
        keeps any substep accepted before the failure, as in the reference."""
        if dt is None:
            dt = self.compute_dt()
        ni = self.n_int
        start = [f[:ni].copy() for f in self._fields()]
        advanced, remaining, halved = 0.0, dt, 0
        while advanced < dt - 1e-15 * dt:
            sub = min(remaining, dt - advanced)
            try:
                self._substep(sub)
            except StateRejected:
                for f, f0 in zip(self._fields(), start):
                    f[:ni] = f0
                halved += 1
                self.retries += 1
                if halved > 12:
                    raise
                advanced, remaining = 0.0, dt / 2**halved
                continue
            advanced += sub
        self.wall_force_series.append((self.t, self.wall_force * self.vol[0]))
        return dt


class EulerianHLLC(EulerianWC):
    """EulerianSolver, ideal-gas branch (eulerian.py:67-85, 269-338, 371-447,
    610-643): limited HLLC flux + energy, ghost kinds incl. the DMR top."""

    def __init__(self, pos, vol, rho, mom, etot, spec, gamma, cfl=0.5, box=None,
                 correction=True, ghosts=None, n_int=None):
        super().__init__(pos, vol, rho, mom, spec, 1.0, 1.0, 0.0, cfl, box, correction, ghosts,
                         n_int)
        self.gamma = gamma
        self.etot = np.array(etot, dtype=float)

    def _fields(self):
        return [self.rho, self.mom, self.etot]

    def eos(self):
        rho = self.rho
        if np.any(rho <= 0.0):
            raise StateRejected("non-positive density")
        v2 = np.sum(self.mom**2, axis=-1) / rho**2
        e = self.etot / rho - 0.5 * v2
        if np.any(e < 0.0):
            raise StateRejected("negative internal energy")
        p = rho * (self.gamma - 1.0) * e
        return p, np.sqrt(self.gamma * p / rho)

    def apply_boundaries(self, t=None):
        g = self.ghosts
        if g is None:
            return
        e0 = self.etot[self.n_int:].copy()
        super().apply_boundaries()
        ni, g0 = self.n_int, self.n_int
        kind = np.asarray(g.kind)
        src = np.asarray(g.src, dtype=np.int64)
        rho, etot = self.rho, self.etot
        etot[g0:] = e0
        for k in (0, 1, 2):
            m = kind == k
            if np.any(m):
                etot[g0:][m] = etot[src[m]]
        m = kind == 3
        if np.any(m):
            etot[g0:][m] = np.asarray(g.fixed)[m, 1 + self.d]
        m = kind == 5
        if np.any(m):
            s, nrm = src[m], np.asarray(g.normal)[m]
            lam = np.asarray(g.blend)[m][:, None]
            vs = self.mom[:ni][s] / rho[:ni][s][:, None]
            vn = np.sum(vs * nrm, axis=1, keepdims=True) * nrm
            vg = vs - 2.0 * lam * vn
            etot[g0:][m] = etot[s] - 0.5 * rho[s] * (np.sum(vs**2, axis=1) - np.sum(vg**2, axis=1))
        m = kind == 4
        if np.any(m):
            par = g.dmr
            xs = par["x0"] + (1.0 + 20.0 * t) / math.tan(math.radians(60.0))
            sel = (np.asarray(par["ghost_x"]) < xs).astype(float)[:, None]
            full = sel * np.asarray(par["post"])[None, :] + (1.0 - sel) * np.asarray(par["pre"])[None, :]
            rho[g0:][m] = full[:, 0]
            self.mom[g0:][m] = full[:, 1:1 + self.d]
            etot[g0:][m] = full[:, 1 + self.d]

    def rhs(self):
        p, c = self.eos()
        v = np.ascontiguousarray(self.mom / self.rho[:, None])
        drho = np.empty(self.n)
        detot = np.empty(self.n)
        dmom = np.zeros((self.n, self.d))
        lib().orc_rhs_hllc(self.n_int, self.d, _p(self.nl.starts), _p(self.nl.idx),
                           _p(self.nl.e), _p(self.gwv), _p(self.rho), _p(v),
                           _p(np.ascontiguousarray(p)), _p(np.ascontiguousarray(c)),
                           _p(self.etot), _p(drho), _p(dmom), _p(detot))
        return drho, dmom, detot

    def compute_dt(self):
        _, c = self.eos()
        ni = self.n_int
        speed = c[:ni] + np.linalg.norm(self.mom[:ni] / self.rho[:ni, None], axis=1)
        return self.cfl * self.spec.h / float(speed.max())

    def _substep(self, dt):
        """eulerian.py:610-643 with the energy equation; rejections (rho <= 0,
        e < 0 in any rhs or after the step, NaN flux) restore the substep
        start.  step() (inherited) adds the retry-with-halving."""
        ni = self.n_int
        r0, m0, e0 = self.rho[:ni].copy(), self.mom[:ni].copy(), self.etot[:ni].copy()
        try:
            self.apply_boundaries(self.t)
            drho, dmom, de = self.rhs()
            if not np.all(np.isfinite(dmom[:ni])):
                raise StateRejected("NaN flux")
            self.rho[:ni] = r0 + 0.5 * dt * drho[:ni]
            self.mom[:ni] = m0 + 0.5 * dt * dmom[:ni]
            self.etot[:ni] = e0 + 0.5 * dt * de[:ni]
            self.apply_boundaries(self.t + 0.5 * dt)
            drho, dmom, de = self.rhs()
            if not np.all(np.isfinite(dmom[:ni])):
                raise StateRejected("NaN flux")
            self.rho[:ni] = r0 + dt * drho[:ni]
            self.mom[:ni] = m0 + dt * dmom[:ni]
            self.etot[:ni] = e0 + dt * de[:ni]
            if not np.all(self.rho[:ni] > 0.0):
                raise StateRejected("non-positive density after step")
            self.eos()
        except StateRejected:
            self.rho[:ni], self.mom[:ni], self.etot[:ni] = r0, m0, e0
            raise
        self.t += dt


# ------------------------------------------------------------ TL-SPH
class SolidTL:
    """SolidSystem (tlsph.py:129-206) with SVK stress; law="neo-hookean"
    selects the compressible Neo-Hookean law S = G (I - C^-1) +
    lam ln(J) C^-1 of BASELINE configs 3-4 — NOT reference-backed (the
    reference implements SVK only): a numpy statement of the
    textbook law, checked against its stored-energy derivative in
    tests/test_host_api.py."""

    def __init__(self, X0, rho0, E, nu, spec, dp, fixed=None, correction=True, cfl=0.6,
                 law="svk"):
        self.law = law
        self.X0 = np.ascontiguousarray(X0, dtype=float)
        self.n, self.d = self.X0.shape
        self.spec, self.dp, self.cfl, self.rho0 = spec, dp, cfl, rho0
        self.lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
        self.g = E / (2.0 * (1.0 + nu))
        self.c_s = float(np.sqrt((self.lam + 2.0 * self.g) / rho0))
        vol0 = np.full(self.n, dp**self.d)
        self.nl = build_neighbors(self.X0, spec.kappa * spec.h)
        if correction:
            self.B0 = correction_matrices(self.nl, vol0, spec)[0]
        else:
            self.B0 = np.tile(np.eye(self.d), (self.n, 1, 1))
        self.B0 = np.ascontiguousarray(self.B0)
        self.g0 = np.ascontiguousarray(pair_gradients(self.nl, spec, None) * vol0[self.nl.idx][:, None])
        self.x = self.X0.copy()
        self.v = np.zeros_like(self.X0)
        self.F = np.tile(np.eye(self.d), (self.n, 1, 1))
        self.fixed = np.zeros(self.n, bool) if fixed is None else np.asarray(fixed, bool)
        self.acc = None
        self.t = 0.0

    def _first_pk_b0(self, sl):
        """P B0^T with P = F S, SVK S (tlsph.py:54-65, 160-167), rows sl."""
        eye = np.eye(self.d)
        F = self.F[sl]
        if self.law == "neo-hookean":
            C = np.einsum("nba,nbc->nac", F, F)
            ci = np.linalg.inv(C)
            ln_j = 0.5 * np.log(np.linalg.det(C))
            s = self.g * (eye - ci) + self.lam * ln_j[:, None, None] * ci
        else:
            strain = 0.5 * (np.einsum("nba,nbc->nac", F, F) - eye)
            tr = np.trace(strain, axis1=1, axis2=2)
            s = self.lam * tr[:, None, None] * eye + 2.0 * self.g * strain
        P = np.einsum("nab,nbc->nac", F, s)
        return np.einsum("nab,ncb->nac", P, self.B0[sl])

    def accelerations(self):
        q = np.ascontiguousarray(np.concatenate(_row_chunks(self.n, self._first_pk_b0)))
        acc = np.empty((self.n, self.d))
        lib().orc_tl_accelerations(self.n, self.d, _p(self.nl.starts), _p(self.nl.idx),
                                   _p(self.g0), _p(q), self.rho0, _p(acc))
        acc[self.fixed] = 0.0
        return acc

    def deformation_rates(self):
        dF = np.empty((self.n, self.d, self.d))
        v = np.ascontiguousarray(self.v)
        lib().orc_tl_deformation_rates(self.n, self.d, _p(self.nl.starts), _p(self.nl.idx),
                                       _p(self.g0), _p(v), _p(self.B0), _p(dF))
        return dF

    def stable_dt(self):
        return self.cfl * self.spec.h / (self.c_s + float(np.linalg.norm(self.v, axis=1).max()))

    def step(self, dt=None):
        if dt is None:
            dt = self.stable_dt()
        if self.acc is None:
            self.acc = self.accelerations()
        self.v += 0.5 * dt * self.acc
        self.v[self.fixed] = 0.0
        self.x += dt * self.v
        self.F += dt * self.deformation_rates()
        if not all(_row_chunks(self.n, lambda sl: bool(np.all(np.linalg.det(self.F[sl]) > 0.0)))):
            raise RuntimeError("deformation gradient inverted")
        self.acc = self.accelerations()
        self.v += 0.5 * dt * self.acc
        self.v[self.fixed] = 0.0
        self.t += dt
        return dt
