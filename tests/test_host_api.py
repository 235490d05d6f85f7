"""Host-side API behaviour the reference's own unit tests pin (kernels,
shapes, lattices): known values, input validation, support and ordering
conventions of `paper_2405_05155_b200.kernels` / `.geometry`
(reference pkg/tests/test_kernels.py, test_geometry.py).  CPU only."""

import math

import numpy as np
import pytest

from paper_2405_05155_b200.geometry import (Box3, Circle, Rectangle, SemiCircle, lattice_fill,
                                            sdf_gradient, signed_distance)
from paper_2405_05155_b200.kernels import (FAMILIES, LAGUERRE_GAUSS, WENDLAND, WENDLAND_TRUNCATED,
                                           cutoff_radius, kernel_grad_magnitude, kernel_spec,
                                           kernel_value, tail_mass, unity_integral)


def _unity_by_quadrature(spec, n=10_000):
    surface = {1: 2.0, 2: 2.0 * math.pi, 3: 4.0 * math.pi}[spec.dim]
    cut = cutoff_radius(spec)
    r = (np.arange(n) + 0.5) * (cut / n)
    return float(np.sum(kernel_value(spec, r) * r ** (spec.dim - 1)) * (cut / n) * surface)


def test_kernel_supports_and_normalisation():
    assert kernel_spec(WENDLAND, 1.0, 2).kappa == 2.0
    assert kernel_spec(WENDLAND_TRUNCATED, 1.0, 2).kappa == 1.6
    assert kernel_spec(LAGUERRE_GAUSS, 1.0, 2).kappa == 2.0
    assert kernel_spec(WENDLAND, 1.0, 2).alpha == pytest.approx(7.0 / (4.0 * math.pi))
    assert cutoff_radius(kernel_spec(WENDLAND, 1.3, 2)) == pytest.approx(2.6)
    assert cutoff_radius(kernel_spec(WENDLAND_TRUNCATED, 1.3, 2)) == pytest.approx(2.08)


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_kernel_unity(family, dim):
    """The truncated kernel keeps the standard normalisation: its support
    integral falls short of one by the discarded tail mass."""
    spec = kernel_spec(family, 1.3, dim)
    unity = _unity_by_quadrature(spec)
    expect = 1.0 - tail_mass(dim) if family == WENDLAND_TRUNCATED else 1.0
    assert unity == pytest.approx(expect, abs=1e-5)
    assert unity_integral(spec) == pytest.approx(unity, abs=1e-6)
    if family == WENDLAND_TRUNCATED:
        assert 0.0 < tail_mass(dim) < 0.01


def test_laguerre_gauss_published_constant_is_not_normalised():
    spec = kernel_spec(LAGUERRE_GAUSS, 1.0, 2)
    assert spec.paper_alpha == pytest.approx(3.0 / math.pi)
    assert abs(spec.paper_alpha / spec.alpha - 1.0) > 0.5


def test_kernel_input_validation():
    with pytest.raises(ValueError):
        kernel_spec("gauss", 1.0, 2)
    with pytest.raises(ValueError):
        kernel_spec(WENDLAND, -1.0, 2)
    with pytest.raises(ValueError):
        kernel_spec(WENDLAND, 1.0, 4)
    spec = kernel_spec(WENDLAND, 1.0, 2)
    with pytest.raises(ValueError):
        kernel_value(spec, -0.1)
    with pytest.raises(ValueError):
        kernel_grad_magnitude(spec, -0.1)


def test_kernel_values_and_support():
    sw, tw = kernel_spec(WENDLAND, 1.0, 2), kernel_spec(WENDLAND_TRUNCATED, 1.0, 2)
    assert kernel_value(sw, 0.0) == pytest.approx(7.0 / (4.0 * math.pi), rel=1e-12)
    assert kernel_value(sw, 2.0) == 0.0 and kernel_value(sw, 2.0 + 1e-12) == 0.0
    assert kernel_value(tw, 1.7) == 0.0
    at_cut = sw.alpha * 0.2**4 * 4.2                    # q = 1.6
    assert at_cut == pytest.approx(3.743e-3, abs=2e-6)
    assert kernel_value(sw, 1.6) == pytest.approx(at_cut, rel=1e-12)
    assert kernel_value(tw, 1.6) == pytest.approx(at_cut, rel=1e-12)
    r = np.linspace(0.0, 1.6 * 1.3, 400)
    s13, t13 = kernel_spec(WENDLAND, 1.3, 2), kernel_spec(WENDLAND_TRUNCATED, 1.3, 2)
    assert np.array_equal(kernel_value(s13, r), kernel_value(t13, r))
    assert np.allclose(kernel_grad_magnitude(s13, r), kernel_grad_magnitude(t13, r))
    vals = [kernel_value(kernel_spec(WENDLAND, h, 2), 0.05) for h in (0.1, 0.01, 0.001)]
    assert vals[0] > 0.0 and vals[1] == 0.0 and vals[2] == 0.0


@pytest.mark.parametrize("family", FAMILIES)
def test_kernel_gradient(family):
    spec = kernel_spec(family, 1.0, 2)
    for r in (0.2, 0.5, 1.0, 1.3, 1.55):
        fd = (kernel_value(spec, r + 1e-6) - kernel_value(spec, r - 1e-6)) / 2e-6
        assert kernel_grad_magnitude(spec, r) == pytest.approx(fd, abs=1e-8)
    r = np.linspace(0.0, 2.5, 500)
    g = kernel_grad_magnitude(spec, r)
    assert np.all(g <= 0.0) and np.all(g[r > spec.kappa] == 0.0)
    assert kernel_grad_magnitude(spec, 0.0) == 0.0
    sw = kernel_spec(WENDLAND, 1.0, 2)
    assert kernel_grad_magnitude(sw, 1.0) == pytest.approx(-0.625 * sw.alpha, rel=1e-12)


def test_signed_distances():
    assert signed_distance(Circle(center=(0.0, 0.0), diameter=2.0), (0.0, 0.0)) == \
        pytest.approx(-1.0)
    assert signed_distance(Rectangle(lo=(0.0, 0.0), hi=(1.0, 1.0)), (0.5, 2.0)) == \
        pytest.approx(1.0)
    s = SemiCircle(center=(0.0, 0.0), radius=0.5, flat_normal=(0.0, 1.0))
    assert float(signed_distance(s, (0.0, 0.0))) == pytest.approx(0.0, abs=1e-14)
    assert float(signed_distance(s, (0.0, -0.5))) == pytest.approx(0.0, abs=1e-14)
    assert float(signed_distance(s, (0.0, -0.25))) < 0.0
    assert float(signed_distance(s, (0.0, 0.25))) == pytest.approx(0.25)
    assert float(signed_distance(s, (0.6, 0.1))) == pytest.approx(np.hypot(0.1, 0.1))
    b = Box3(lo=(0, 0, 0), hi=(1, 1, 1))
    assert signed_distance(b, (0.5, 0.5, 0.5)) == pytest.approx(-0.5)
    assert signed_distance(b, (2.0, 0.5, 0.5)) == pytest.approx(1.0)
    c = Circle(center=(0.25, -0.5), diameter=1.5)
    rng = np.random.default_rng(0)
    for x, y in rng.uniform(-2, 2, size=(30, 2)):
        assert signed_distance(c, (x, y)) == pytest.approx(np.hypot(x - 0.25, y + 0.5) - 0.75,
                                                          abs=1e-12)
    g = sdf_gradient(Circle(center=(0.0, 0.0), diameter=2.0), [(0.5, 0.0), (0.0, -0.3)])
    assert g[0] == pytest.approx([1.0, 0.0], abs=1e-6)
    assert g[1] == pytest.approx([0.0, -1.0], abs=1e-6)


def test_invalid_shapes():
    with pytest.raises(ValueError):
        Circle(center=(0, 0), diameter=-1.0)
    with pytest.raises(ValueError):
        Rectangle(lo=(0, 0), hi=(0, 1))
    with pytest.raises(ValueError):
        SemiCircle(center=(0, 0), radius=0.5, flat_normal=(0, 2.0))
    with pytest.raises(ValueError):
        Box3(lo=(0, 0), hi=(1, 1))
    with pytest.raises(ValueError):
        signed_distance(Circle(center=(0, 0), diameter=1.0), (np.nan, 0.0))


def test_lattice_fill():
    pts = lattice_fill(Rectangle(lo=(0, 0), hi=(1, 1)), 0.25)
    assert pts.shape == (16, 2)
    assert sorted(set(np.round(pts[:, 0], 12))) == [0.125, 0.375, 0.625, 0.875]
    assert lattice_fill(Box3(lo=(0, 0, 0), hi=(1, 1, 1)), 0.5).shape == (8, 3)
    circle = Circle(center=(0.0, 0.0), diameter=2.0)
    axes = -1.0 + (np.arange(10) + 0.5) * 0.2
    xx, yy = np.meshgrid(axes, axes)
    assert lattice_fill(circle, 0.2).shape[0] == int((np.hypot(xx, yy) < 1.0).sum())
    off = Circle(center=(0.3, -0.2), diameter=1.4)
    assert np.all(off.signed_distance(lattice_fill(off, 0.07)) < 0.0)
    assert lattice_fill(circle, 0.025).shape[0] / lattice_fill(circle, 0.1).shape[0] == \
        pytest.approx(16.0, rel=0.05)
    with pytest.raises(ValueError):
        lattice_fill(Circle(center=(0, 0), diameter=0.1), 0.5)
    a = lattice_fill(Rectangle(lo=(0, 0), hi=(1, 1)), 0.2)
    assert np.array_equal(a, lattice_fill(Rectangle(lo=(0, 0), hi=(1, 1)), 0.2))
    assert a[0] == pytest.approx([0.1, 0.1]) and a[1] == pytest.approx([0.1, 0.3])


def test_neo_hookean_stress_is_the_energy_derivative():
    """The optional compressible Neo-Hookean law (BASELINE configs 3-4; not in
    the reference): S = 2 dW/dC for W = G/2 (tr C - d) - G ln J + lam/2 ln^2 J,
    checked by central differences on random deformations; small strains
    agree with SVK to first order."""
    from paper_2405_05155_b200.tlsph import NEO_HOOKEAN, Material, pk2_stress

    mat = Material(rho0=1100.0, E=1.7e7, nu=0.45, law=NEO_HOOKEAN)
    lam, g = mat.lame
    rng = np.random.default_rng(4)

    def energy(C):
        d = C.shape[0]
        ln_j = 0.5 * np.log(np.linalg.det(C))
        return 0.5 * g * (np.trace(C) - d) - g * ln_j + 0.5 * lam * ln_j**2

    for d in (2, 3):
        for _ in range(5):
            F = np.eye(d) + 0.2 * rng.standard_normal((d, d))
            C = F.T @ F
            S = pk2_stress(F, mat)
            num = np.zeros((d, d))
            eps = 1e-6
            for a in range(d):
                for b in range(d):
                    dC = np.zeros((d, d))
                    dC[a, b] += eps / 2
                    dC[b, a] += eps / 2
                    num[a, b] = 2.0 * (energy(C + dC) - energy(C - dC)) / (2 * eps)
            assert np.allclose(S, num, rtol=1e-6, atol=1e-6 * np.abs(S).max())
        F = np.eye(d) + 1e-7 * rng.standard_normal((d, d))
        svk = pk2_stress(F, Material(rho0=1100.0, E=1.7e7, nu=0.45))
        assert np.allclose(pk2_stress(F, mat), svk, rtol=1e-5, atol=1e-5 * np.abs(svk).max())
    with pytest.raises(ValueError):
        Material(rho0=1.0, E=1.0, nu=0.3, law="mooney")
