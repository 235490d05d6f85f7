"""The five BASELINE.json configurations as seeded synthetic inputs.

None of them is a case shipped with the reference, so each
is a thin constructor over the reference primitives' conventions (SURVEY §8(d)
and Appendix B):

  C1  perturbed periodic lattice, Laguerre-Gauss relaxation, density sums
  C2  2D Taylor-Green vortex, WC Eulerian (template: cases.py:370-388)
  C3  2D clamped cantilever plate, TL-SPH       (template: cases.py:437-461)
  C4  3D twisting column, TL-SPH                (cases.py:437-461)
  C5  3D Taylor-Green vortex, WC Eulerian

Every builder returns plain numpy inputs in lattice_points order, so the
same dictionaries feed the GPU engine, the oracle and the golden-fixture
script.  `scale` arguments shrink a config for parity tests (the particle
spacing changes, the physics and h/dp ratios do not).
"""

from __future__ import annotations

import math

import numpy as np

from .geometry import lattice_points
from .kernels import LAGUERRE_GAUSS, WENDLAND, WENDLAND_TRUNCATED, kernel_spec

FAMILY = {"1.6h": WENDLAND_TRUNCATED, "2h": WENDLAND}


def c1_relax(seed: int = 0, n_side: int = 100, perturb: float = 0.2):
    """C1: unit square, periodic, dx = 1/n_side, uniform(-0.2dx, 0.2dx) jitter,
    h = 1.3dx, LG relaxation for 100 updates (step_scale 0.2, p0 = rho0 = 1)."""
    dx = 1.0 / n_side
    pos = lattice_points((0.0, 0.0), (1.0, 1.0), dx)
    rng = np.random.default_rng(seed)
    pos = pos + rng.uniform(-perturb * dx, perturb * dx, size=pos.shape)
    pos %= 1.0
    h = 1.3 * dx
    return {
        "name": "c1_relax", "pos": pos, "box": (1.0, 1.0), "dp": dx, "h": h,
        "relax_spec": kernel_spec(LAGUERRE_GAUSS, h, 2), "n_updates": 100,
        "vol": dx * dx, "p0": 1.0, "rho0": 1.0, "step_scale": 0.2,
    }


def _tgv2d_fields(pos, c):
    x, y = pos[:, 0], pos[:, 1]
    u = -np.cos(2.0 * np.pi * x) * np.sin(2.0 * np.pi * y)
    v = np.sin(2.0 * np.pi * x) * np.cos(2.0 * np.pi * y)
    p = -0.25 * (np.cos(4.0 * np.pi * x) + np.cos(4.0 * np.pi * y))
    rho = 1.0 + p / c**2
    return rho, np.column_stack([rho * u, rho * v])


def c2_tgv2d(kernel: str = "1.6h", n_side: int = 200, steps: int = 1000):
    """C2: [0,1]^2 periodic, rho0 = U = 1, c0 = 10, Re = 100 (mu = 0.01),
    acoustic CFL 0.25, B_i on."""
    dp = 1.0 / n_side
    pos = lattice_points((0.0, 0.0), (1.0, 1.0), dp)
    c = 10.0
    rho, mom = _tgv2d_fields(pos, c)
    return {
        "name": "c2_tgv2d", "pos": pos, "box": (1.0, 1.0), "dp": dp,
        "spec": kernel_spec(FAMILY[kernel], 1.3 * dp, 2),
        "vol": np.full(pos.shape[0], dp * dp), "rho": rho, "mom": mom,
        "c_art": c, "rho0": 1.0, "mu": 0.01, "cfl": 0.25, "steps": steps,
    }


def _tgv3d_fields(pos, c):
    x, y, z = pos[:, 0], pos[:, 1], pos[:, 2]
    u = np.sin(x) * np.cos(y) * np.cos(z)
    v = -np.cos(x) * np.sin(y) * np.cos(z)
    w = np.zeros_like(u)
    p = (1.0 / 16.0) * (np.cos(2.0 * x) + np.cos(2.0 * y)) * (np.cos(2.0 * z) + 2.0)
    rho = 1.0 + p / c**2
    return rho, np.column_stack([rho * u, rho * v, rho * w])


def c5_tgv3d(kernel: str = "1.6h", n_side: int = 256, steps: int = 200):
    """C5: periodic [0, 2pi]^3, rho0 = U = 1, c0 = 10, Re = 1600
    (mu = 1/1600), CFL 0.25 (not stated in BASELINE)."""
    L = 2.0 * math.pi
    dp = L / n_side
    pos = lattice_points((0.0, 0.0, 0.0), (L, L, L), dp)
    c = 10.0
    rho, mom = _tgv3d_fields(pos, c)
    return {
        "name": "c5_tgv3d", "pos": pos, "box": (L, L, L), "dp": dp,
        "spec": kernel_spec(FAMILY[kernel], 1.3 * dp, 3),
        "vol": np.full(pos.shape[0], dp**3), "rho": rho, "mom": mom,
        "c_art": c, "rho0": 1.0, "mu": 1.0 / 1600.0, "cfl": 0.25, "steps": steps,
    }


def _cantilever_mode(xi, length):
    """First clamped-free bending mode, kL = 1.875 (x measured from the clamp)."""
    k = 1.875 / length
    kl = k * length
    a = (math.cosh(kl) + math.cos(kl)) / (math.sinh(kl) + math.sin(kl))
    return (np.cosh(k * xi) - np.cos(k * xi)) - a * (np.sinh(k * xi) - np.sin(k * xi))


def c3_plate(kernel: str = "1.6h", dp: float = 0.001, steps: int = 2000, vf: float = 0.05):
    """C3: plate L = 0.2, H = 0.02 plus a 0.06 clamp (x < 0), H/dp = 20,
    rho0 = 1000, E = 2e6, nu = 0.3975, h = 1.15 dp.  v_y = vf c_s f(x)/f(L)
    with f the first clamped-free mode (normalisation recorded in DESIGN.md)."""
    from .tlsph import Material

    L, H, clamp = 0.2, 0.02, 0.06
    X0 = lattice_points((-clamp, 0.0), (L, H), dp)
    fixed = X0[:, 0] < 0.0
    mat = Material(rho0=1000.0, E=2.0e6, nu=0.3975)
    xi = np.maximum(X0[:, 0], 0.0)
    v = np.zeros_like(X0)
    v[:, 1] = vf * mat.sound_speed * _cantilever_mode(xi, L) / _cantilever_mode(np.array(L), L)
    v[fixed] = 0.0
    return {
        "name": "c3_plate", "X0": X0, "dp": dp, "fixed": fixed, "v0": v, "material": mat,
        "spec": kernel_spec(FAMILY[kernel], 1.15 * dp, 2), "cfl": 0.6, "steps": steps,
    }


def c4_column(kernel: str = "1.6h", n_width: int = 68, steps: int = 500, omega0: float = 100.0):
    """C4: column 1 x 6 x 1, dp = 1/n_width (68 -> 1,886,592 particles),
    clamp y < kappa h (cases.py:446), rho0 = 1100, E = 1.7e7, nu = 0.45,
    omega(y) = 100 sin(pi y / 12) about the long axis, h = 1.15 dp."""
    from .tlsph import Material, TWIST, init_case_velocity

    dp = 1.0 / n_width
    X0 = lattice_points((-0.5, 0.0, -0.5), (0.5, 6.0, 0.5), dp)
    spec = kernel_spec(FAMILY[kernel], 1.15 * dp, 3)
    fixed = X0[:, 1] < spec.kappa * spec.h
    v = init_case_velocity(TWIST, X0, length=6.0, omega0=omega0)
    v[fixed] = 0.0
    return {
        "name": "c4_column", "X0": X0, "dp": dp, "fixed": fixed, "v0": v,
        "material": Material(rho0=1100.0, E=1.7e7, nu=0.45), "spec": spec, "cfl": 0.6,
        "steps": steps,
    }


def density_specs(h: float, dim: int = 2):
    """Wendland truncated (1.6h) and standard (2h) specs for density sums."""
    return {k: kernel_spec(f, h, dim) for k, f in FAMILY.items()}
