"""Pin the CPU oracle to the reference (CPU only, no GPU needed).

The oracle (oracle/) is the checker of every GPU parity test, so it is
trusted only after matching (a) golden vectors produced by the reference
package itself (tests/golden/make_golden.py) and (b) every known value the
reference's own unit tests assert for the hot path (pkg/tests/*).
"""

import hashlib

import numpy as np
import pytest

from conftest import checkpoints
from oracle import oracle as O
from paper_2405_05155_b200 import configs
from paper_2405_05155_b200.geometry import lattice_points
from paper_2405_05155_b200.kernels import kernel_spec


def digest(nl):
    h = hashlib.sha256()
    for a in (nl.starts, nl.idx, nl.r, nl.e):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


NEIGHBOR_CASES = ["random500", "periodic300", "random3d_200", "lattice_sw", "lattice_tw",
                  "lattice3d", "periodic_lattice8", "exact_cutoff", "random1d_100"]


@pytest.mark.parametrize("case", NEIGHBOR_CASES)
def test_oracle_csr_byte_identical(gold, case):
    g = gold("neighbors")
    box = g[f"{case}__box"]
    nl = O.build_neighbors(g[f"{case}__pos"], float(g[f"{case}__cutoff"]),
                           box if box.size else None)
    assert np.array_equal(nl.starts, g[f"{case}__starts"])
    assert np.array_equal(nl.idx, g[f"{case}__idx"])
    assert np.array_equal(nl.r, g[f"{case}__r"])
    assert np.array_equal(nl.e, g[f"{case}__e"])
    assert digest(nl) == str(g[f"{case}__digest"])


def test_oracle_lattice_counts():
    # pkg/tests/test_neighbors.py:38-45
    pos = lattice_points((0, 0), (9, 9), 1.0)
    c = np.argmin(np.linalg.norm(pos - 4.5, axis=1))
    assert O.build_neighbors(pos, 2.6).counts[c] == 20
    assert O.build_neighbors(pos, 2.08).counts[c] == 12


def test_oracle_brute_force_periodic(rng):
    # pkg/tests/test_neighbors.py:68-81 with the O(N^2) minimum-image oracle
    pos = rng.uniform(0, 1, size=(300, 2))
    box = np.array([1.0, 1.0])
    nl = O.build_neighbors(pos, 0.13, box)
    want = set()
    for i in range(300):
        d = pos[i] - pos
        d -= np.round(d / box) * box
        r = np.linalg.norm(d, axis=1)
        want |= {(i, int(j)) for j in np.where((r <= 0.13) & (r > 0))[0]}
    got = {(i, int(j)) for i in range(nl.n) for j in nl.idx[nl.starts[i]:nl.starts[i + 1]]}
    assert got == want


FAMS = ["wendland", "wendland_truncated", "laguerre_gauss"]


@pytest.mark.parametrize("fam", FAMS)
def test_oracle_operators(gold, fam):
    g = gold("operators")
    spec = kernel_spec(fam.replace("_", "-"), 0.05, 2)
    nl = O.build_neighbors(g["pos"], 2.0 * spec.h)
    vols = g["vols"]
    # the C loops are the reference loops: bit-identical
    assert np.array_equal(O.sph_unity_sum(nl, vols, spec), g[f"{fam}__unity"])
    assert np.array_equal(O.relax_accelerations(nl, vols, spec, 1.3, 0.9), g[f"{fam}__accel"])
    assert np.array_equal(O.moment_matrices(nl, vols, spec), g[f"{fam}__moments"])
    b, det, nreg = O.correction_matrices(nl, vols, spec)
    np.testing.assert_allclose(b, g[f"{fam}__B"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(det, g[f"{fam}__det"], rtol=1e-12, atol=1e-14)
    assert nreg == int(g[f"{fam}__nreg"])
    assert np.array_equal(O.pair_gradients(nl, spec, g[f"{fam}__B"]), g[f"{fam}__gw"])
    assert np.array_equal(O.pair_gradients(nl, spec, None), g[f"{fam}__gw0"])


def test_oracle_correction_known_values():
    # pkg/tests/test_correction.py:22-48, 78-81
    for fam, m00, bscale in (("wendland", -0.9739, 1.0268), ("wendland-truncated", -0.9204, 1.0864)):
        pos = lattice_points((0, 0), (13.0, 13.0), 1.0)
        spec = kernel_spec(fam, 1.3, 2)
        nl = O.build_neighbors(pos, spec.kappa * spec.h)
        c = int(np.argmin(np.linalg.norm(pos - 6.5, axis=1)))
        m = O.moment_matrices(nl, np.ones(len(pos)), spec)[c]
        assert m[0, 0] == pytest.approx(m00, abs=2e-4)
        assert m[0, 1] == pytest.approx(0.0, abs=1e-12)
        b = O.correction_matrices(nl, np.ones(len(pos)), spec)[0][c]
        assert b[0, 0] == pytest.approx(bscale, abs=2e-3)
    pos = lattice_points((0, 0), (9.0, 9.0), 1.0)
    spec = kernel_spec("wendland", 1.3, 2)
    nl = O.build_neighbors(pos, spec.kappa * spec.h)
    c = int(np.argmin(np.linalg.norm(pos - 4.5, axis=1)))
    assert O.correction_matrices(nl, np.ones(len(pos)), spec)[1][c] == pytest.approx(0.9485, abs=1e-3)


def test_oracle_c1_relaxation(gold):
    g = gold("c1_relax")
    c1 = configs.c1_relax(seed=0)
    assert np.array_equal(c1["pos"], g["pos0"])
    spec = kernel_spec("laguerre-gauss", c1["h"], 2)
    # one update is the reference bit for bit (same libm exp on this host)
    pos1, res1 = O.relax_steps(c1["pos"], spec, c1["box"], c1["dp"], 1)
    assert np.array_equal(pos1, g["pos1"])
    assert digest(O.build_neighbors(g["pos1"], spec.kappa * spec.h, c1["box"])) == str(g["digests"][1])
    np.testing.assert_allclose(res1, g["residuals"][:2], rtol=1e-13)


@pytest.mark.slow
def test_oracle_c1_100_updates(gold):
    g = gold("c1_relax")
    c1 = configs.c1_relax(seed=0)
    spec = kernel_spec("laguerre-gauss", c1["h"], 2)
    pos, res = O.relax_steps(c1["pos"], spec, c1["box"], c1["dp"], 100)
    np.testing.assert_allclose(res, g["residuals"], rtol=1e-12)
    assert np.array_equal(pos, g["pos100"])
    for key, tag in (("1.6h", "1p6h"), ("2h", "2h")):
        ds = configs.density_specs(c1["h"])[key]
        nl = O.build_neighbors(pos, ds.kappa * ds.h, c1["box"])
        assert digest(nl) == str(g[f"digest_{tag}"])
        assert np.array_equal(O.sph_unity_sum(nl, np.full(len(pos), c1["vol"]), ds), g[f"rho_{tag}"])


@pytest.mark.parametrize("label,builder", [("c2_tgv2d", configs.c2_tgv2d),
                                           ("c5_tgv3d", configs.c5_tgv3d)])
@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_oracle_wc_tgv(gold, label, builder, key):
    g = gold(label)
    tag = key.replace(".", "p")
    cfg = builder(kernel=key, n_side=int(g["n_side"]))
    s = O.EulerianWC(cfg["pos"], cfg["vol"], cfg["rho"], cfg["mom"], cfg["spec"], cfg["c_art"],
                     cfg["rho0"], cfg["mu"], cfg["cfl"], cfg["box"])
    assert digest(s.nl) == str(g[f"{tag}__digest"])
    drho, dmom = s.rhs()
    np.testing.assert_allclose(drho, g[f"{tag}__drho0"], rtol=0, atol=1e-12 * np.abs(drho).max())
    np.testing.assert_allclose(dmom, g[f"{tag}__dmom0"], rtol=0, atol=1e-12 * np.abs(dmom).max())
    from paper_2405_05155_b200.approx import l2_error

    steps = int(g["steps"])
    marks = checkpoints(g, tag, "rho")
    assert marks[0] == 1 and marks[-1] == steps and (steps < 100 or 100 in marks)
    dts = []
    for k in range(1, steps + 1):
        dts.append(s.step())
        if k in marks:
            tol = 1e-13 if k == 1 else 1e-10
            assert l2_error(s.rho, g[f"{tag}__rho{k}"]) < tol
            assert l2_error(s.mom, g[f"{tag}__mom{k}"]) < tol
    np.testing.assert_allclose(dts, g[f"{tag}__dts"], rtol=1e-13)


@pytest.mark.parametrize("key", ["1.6h", "2h"])
@pytest.mark.parametrize("mult", [20, 40])
def test_oracle_retry_with_halving(gold, key, mult):
    """Forced halving (eulerian.py:562-608): per-step state, t and the
    cumulative retry count against the reference's own run."""
    from paper_2405_05155_b200.approx import l2_error

    g = gold("retry")
    tag = f"{key.replace('.', 'p')}_x{mult}"
    cfg = configs.c2_tgv2d(kernel=key, n_side=int(g["n_side"]))
    s = O.EulerianWC(cfg["pos"], cfg["vol"], cfg["rho"], cfg["mom"], cfg["spec"], cfg["c_art"],
                     cfg["rho0"], cfg["mu"], cfg["cfl"], cfg["box"])
    dt = float(g[f"{tag}__dt"])
    for k in range(1, 6):
        s.step(dt)
        assert s.retries == int(g[f"{tag}__retries"][k - 1])
        assert s.t == pytest.approx(float(g[f"{tag}__t"][k - 1]), rel=1e-14)
        assert l2_error(s.rho, g[f"{tag}__rho{k}"]) < 1e-12
        assert l2_error(s.mom, g[f"{tag}__mom{k}"]) < 1e-12


@pytest.mark.parametrize("label,builder,kwargs", [("c3_plate", configs.c3_plate, {"dp": 0.002}),
                                                  ("c4_column", configs.c4_column, {"n_width": 6})])
@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_oracle_tl(gold, label, builder, kwargs, key):
    g = gold(label)
    tag = key.replace(".", "p")
    cfg = builder(kernel=key, **kwargs)
    m = cfg["material"]
    s = O.SolidTL(cfg["X0"], m.rho0, m.E, m.nu, cfg["spec"], cfg["dp"], cfg["fixed"], True, cfg["cfl"])
    assert digest(s.nl) == str(g[f"{tag}__digest"])
    np.testing.assert_allclose(s.B0, g[f"{tag}__B0"], rtol=1e-12, atol=1e-12)
    s.v = cfg["v0"].copy()
    steps = int(g["steps"])
    from paper_2405_05155_b200.approx import l2_error

    marks = checkpoints(g, tag, "x")
    assert marks[0] == 1 and marks[-1] == steps and 100 in marks
    dts = []
    for k in range(1, steps + 1):
        dts.append(s.step())
        if k in marks:
            tol = 1e-12 if k == 1 else 1e-9
            assert l2_error(s.x, g[f"{tag}__x{k}"]) < tol
            assert l2_error(s.v, g[f"{tag}__v{k}"]) < tol
            assert l2_error(s.F, g[f"{tag}__F{k}"]) < tol
    np.testing.assert_allclose(dts, g[f"{tag}__dts"], rtol=1e-13)


class _Ghosts:
    def __init__(self, g, tag):
        self.kind, self.src = g[f"{tag}__kind"], g[f"{tag}__src"]
        self.normal, self.wall_v = g[f"{tag}__normal"], g[f"{tag}__wall_v"]
        self.fixed, self.blend = g[f"{tag}__fixed"], g[f"{tag}__blend"]


@pytest.mark.parametrize("case", ["cavity", "mixed"])
@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_oracle_ghost_layers(gold, case, key):
    """Ghost frames of cases.build_rect_case (wall / mirror / blend / fixed /
    copy) through the oracle's apply_boundaries restatement."""
    from paper_2405_05155_b200.approx import l2_error

    g = gold(f"ghosts_{case}")
    tag = key.replace(".", "p")
    pos, ni = g[f"{tag}__pos"], int(g["n_int"])
    dp = 1.0 / 20
    spec = kernel_spec(configs.FAMILY[key], 1.3 * dp, 2)
    n = pos.shape[0]
    s = O.EulerianWC(pos, np.full(n, dp * dp), g["rho_init"], g["mom_init"], spec, 10.0, 1.0,
                     0.0025, 0.5, None, ghosts=_Ghosts(g, tag), n_int=ni)
    for k in range(1, 51):
        s.step()
        if k in (1, 50):
            tol = 1e-13 if k == 1 else 1e-10
            assert l2_error(s.rho[:ni], g[f"{tag}__rho{k}"]) < tol
            assert l2_error(s.mom[:ni], g[f"{tag}__mom{k}"]) < tol


class _DmrGhosts(_Ghosts):
    def __init__(self, g, tag):
        super().__init__(g, tag)
        self.dmr = {"x0": float(g[f"{tag}__dmr_x0"]), "ghost_x": g[f"{tag}__dmr_ghost_x"],
                    "post": g[f"{tag}__dmr_post"], "pre": g[f"{tag}__dmr_pre"]}


def oracle_dmr(g, tag, key):
    """cases.build_dmr at dp = 1/16 through the oracle's HLLC restatement."""
    dp = 1.0 / 16
    spec = kernel_spec(configs.FAMILY[key], 1.3 * dp, 2)
    pos = g[f"{tag}__pos"]
    n = pos.shape[0]
    return O.EulerianHLLC(pos, np.full(n, dp * dp), g[f"{tag}__rho_init"], g[f"{tag}__mom_init"],
                          g[f"{tag}__etot_init"], spec, 1.4, 0.5, None,
                          ghosts=_DmrGhosts(g, tag), n_int=int(g[f"{tag}__n_int"]))


@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_oracle_hllc_dmr(gold, key):
    """Compressible HLLC + energy with the double-Mach-reflection ghost frame
    (eulerian.py:269-338 flux, 610-643 boundaries; cases.py build_dmr)."""
    from paper_2405_05155_b200.approx import l2_error

    g = gold("hllc_dmr")
    tag = key.replace(".", "p")
    s = oracle_dmr(g, tag, key)
    ni = s.n_int
    drho, dmom, de = s.rhs()     # initial ghost states, as built (no boundary pass yet)
    assert l2_error(drho[:ni], g[f"{tag}__drho0"][:ni]) < 1e-13
    assert l2_error(dmom[:ni], g[f"{tag}__dmom0"][:ni]) < 1e-13
    assert l2_error(de[:ni], g[f"{tag}__de0"][:ni]) < 1e-13
    dts = []
    for k in range(1, 21):
        dts.append(s.step())
        if k in (1, 20):
            tol = 1e-13 if k == 1 else 1e-10
            assert l2_error(s.rho[:ni], g[f"{tag}__rho{k}"]) < tol
            assert l2_error(s.mom[:ni], g[f"{tag}__mom{k}"]) < tol
            assert l2_error(s.etot[:ni], g[f"{tag}__etot{k}"]) < tol
    np.testing.assert_allclose(dts, g[f"{tag}__dts"], rtol=1e-10)


def oracle_cylinder(g, tag, key):
    """cases.build_cylinder (reduced: D = 1, 5 x 3 box, dp = 0.1, Re 20)."""
    dp = 0.1
    spec = kernel_spec(configs.FAMILY[key], 1.3 * dp, 2)
    pos = g[f"{tag}__pos"]
    n = pos.shape[0]
    return O.EulerianWC(pos, np.full(n, dp * dp), g[f"{tag}__rho_init"], g[f"{tag}__mom_init"],
                        spec, 10.0, 1.0, float(g[f"{tag}__mu"]), 0.5, None,
                        ghosts=_CylGhosts(g, tag), n_int=int(g[f"{tag}__n_int"]),
                        wall_tag=g[f"{tag}__wall_tag"])


class _CylGhosts(_Ghosts):
    def __init__(self, g, tag):
        self.kind, self.src = g[f"{tag}__kind"], g[f"{tag}__src"]
        self.normal, self.wall_v = g[f"{tag}__normal"], g[f"{tag}__wall_v"]
        self.fixed, self.blend = g[f"{tag}__fixed"], None


@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_oracle_cylinder_wall_force(gold, key):
    """Flow past a cylinder: in-body wall ghosts (G_WALL, KD-tree mirrored
    sources), fixed far field, and the wall-force series (eulerian.py:262-264,
    605-606) that the drag/lift coefficients come from."""
    from paper_2405_05155_b200.approx import l2_error

    g = gold("cylinder")
    tag = key.replace(".", "p")
    s = oracle_cylinder(g, tag, key)
    ni = s.n_int
    dts = [s.step() for _ in range(30)]
    assert l2_error(s.rho[:ni], g[f"{tag}__rho30"]) < 1e-10
    assert l2_error(s.mom[:ni], g[f"{tag}__mom30"]) < 1e-10
    np.testing.assert_allclose(dts, g[f"{tag}__dts"], rtol=1e-12)
    wf = np.array([w for _, w in s.wall_force_series])
    np.testing.assert_allclose([t for t, _ in s.wall_force_series], g[f"{tag}__wf_t"], rtol=1e-12)
    assert l2_error(wf, g[f"{tag}__wf"]) < 1e-10


_ORC_SHAPES = {
    "circle": O.Shape("circle", center=(0.0, 0.0), radius=1.0),
    "semicircle": O.Shape("semicircle", center=(0.0, 0.0), radius=0.5, normal=(0.0, 1.0)),
    "rectangle": O.Shape("rectangle", lo=(0.0, 0.0), hi=(1.0, 0.5)),
    "ball": O.Shape("circle", center=(0.1, 0.2, 0.3), radius=0.5),
    "box3": O.Shape("rectangle", lo=(0.0, 0.0, 0.0), hi=(1.0, 0.5, 0.25)),
}


@pytest.mark.parametrize("name", sorted(_ORC_SHAPES))
def test_oracle_sdf(gold, name):
    """Signed distances and central-difference normals (geometry.py:16-147)."""
    g = gold("relax_shapes")
    s = _ORC_SHAPES[name]
    x = g[f"sdf_{name}__x"]
    np.testing.assert_allclose(s.signed_distance(x), g[f"sdf_{name}__sd"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(s.gradient(x), g[f"sdf_{name}__grad"], rtol=0, atol=1e-9)


def test_oracle_wall_confinement(gold):
    """Planar kernel integral w2(s) (relaxation.py:92-117), interpolated."""
    g = gold("relax_shapes")
    for fam, hr, dim in (("wendland", 1.3, 2), ("laguerre-gauss", 1.1, 2), ("wendland", 1.3, 3)):
        spec = kernel_spec(fam, hr * 0.1, dim)
        w = O.wall_confinement(spec, g[f"wall_{fam}_{dim}__depth"])
        np.testing.assert_array_equal(w, g[f"wall_{fam}_{dim}__w2"])


@pytest.mark.parametrize("tag,shape,fam", [("circle_w", "circle", "wendland"),
                                           ("circle_lg", "circle", "laguerre-gauss"),
                                           ("semicircle_lg", "semicircle", "laguerre-gauss"),
                                           ("rectangle_w", "rectangle", "wendland")])
def test_oracle_shape_relaxation(gold, tag, shape, fam):
    """Shape-bounded relax(): confinement + projection, 40 updates."""
    g = gold("relax_shapes")
    dp, hr, ss = g[f"{tag}__params"]
    spec = kernel_spec(fam, hr * dp, 2)
    s = _ORC_SHAPES[shape]
    np.testing.assert_array_equal(s.lattice_fill(dp), g[f"{tag}__pos0"])
    pos, res, best = O.relax_shape(s, spec, dp, 40, step_scale=ss)
    assert best == int(g[f"{tag}__meta"][1])
    np.testing.assert_allclose(res, g[f"{tag}__residuals"], rtol=1e-9)
    np.testing.assert_allclose(pos, g[f"{tag}__positions"], rtol=0, atol=1e-10)


def test_oracle_weak_gradient(gold):
    """Weak-form gradient, plain and corrected (approx.py:61-86)."""
    g = gold("error_study")
    pos = g["wg__pos"]
    spec = kernel_spec("wendland", 0.13, 2)
    nl = O.build_neighbors(pos, spec.kappa * spec.h)
    vols = np.full(pos.shape[0], 0.008)
    f = np.exp(-(pos[:, 0] ** 2) / 0.1)
    np.testing.assert_allclose(O.weak_gradient(nl, f, vols, spec), g["wg__plain"], rtol=0,
                               atol=1e-12)
    b = O.correction_matrices(nl, vols, spec)[0]
    np.testing.assert_allclose(O.weak_gradient(nl, f, vols, spec, b), g["wg__corrected"], rtol=0,
                               atol=1e-11)


@pytest.mark.parametrize("fam", ["wendland", "wendland-truncated", "laguerre-gauss"])
def test_oracle_circle_study_errors(gold, fam):
    """Unity and gradient errors of the circle study on the lattice
    distribution (approx.py:148-192), oracle operators + study glue."""
    g = gold("error_study")
    key = fam.replace("-", "_")
    circle = O.Shape("circle", center=(0.0, 0.0), radius=1.0)
    for k, dp in enumerate((0.2, 0.1)):
        pos = circle.lattice_fill(dp)
        spec = kernel_spec(fam, 1.3 * dp, 2)
        vols = np.full(pos.shape[0], dp * dp)
        mask = np.linalg.norm(pos, axis=1) <= 1.0 - 2.0 * 1.3 * dp
        u = O.sph_unity_sum(O.build_neighbors(pos, 2.0 * spec.h), vols, spec)
        np.testing.assert_allclose(np.linalg.norm(u[mask] - 1.0) / np.sqrt(mask.sum()),
                                   g[f"unity__{key}__{k}"], rtol=1e-12)
        nl = O.build_neighbors(pos, spec.kappa * spec.h)
        for corr in (False, True):
            b = O.correction_matrices(nl, vols, spec)[0] if corr else None
            grad = O.weak_gradient(nl, np.exp(-(pos[:, 0] ** 2) / 0.1), vols, spec, b)
            ana = -(20.0 * pos[mask, 0]) * np.exp(-(pos[mask, 0] ** 2) / 0.1)
            err = np.linalg.norm(grad[mask, 0] - ana) / np.linalg.norm(ana)
            np.testing.assert_allclose(err, g[f"grad__{key}__{k}__{int(corr)}"], rtol=1e-9)


@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_oracle_hllc_retry_with_halving(gold, key):
    """Forced halving on the HLLC path (DMR at 8x the CFL step): retries, t
    and (rho, mom, E) after each of 6 steps against the reference."""
    from paper_2405_05155_b200.approx import l2_error

    g = gold("retry_hllc")
    tag = key.replace(".", "p")
    s = oracle_dmr(gold("hllc_dmr"), tag, key)
    ni = s.n_int
    for k in range(1, 7):
        s.step(float(g[f"{tag}__dt"][k - 1]))
        assert s.retries == int(g[f"{tag}__retries"][k - 1])
        assert s.t == pytest.approx(float(g[f"{tag}__t"][k - 1]), rel=1e-14)
        for f in ("rho", "mom", "etot"):
            assert l2_error(getattr(s, f)[:ni], g[f"{tag}__{f}{k}"]) < 1e-11, (k, f)
