"""Case builders (cases.py) against fixtures made by the reference's own
builders (tests/golden/make_golden.py): ghost frames, sources, prescribed
states, the DMR and cylinder set-ups.  Host-only tests build the frames;
the `gpu` tests also construct the solvers and step them."""

import numpy as np
import pytest

from paper_2405_05155_b200 import cases, configs
from paper_2405_05155_b200.approx import l2_error
from paper_2405_05155_b200.eulerian import (G_BLEND_MIRROR, G_COPY, G_FIXED, G_MIRROR, G_WALL,
                                            WEAKLY_COMPRESSIBLE, EosParams)
from paper_2405_05155_b200.kernels import kernel_spec

SIDES = {
    "cavity": lambda: {"y+": cases.SideSpec(G_WALL, wall_v=(1.0, 0.0)),
                       "y-": cases.SideSpec(G_WALL), "x-": cases.SideSpec(G_WALL),
                       "x+": cases.SideSpec(G_WALL)},
    "mixed": lambda: {"y+": cases.SideSpec(G_WALL, wall_v=(0.5, 0.0)),
                      "y-": cases.SideSpec(G_MIRROR),
                      "x-": cases.SideSpec(G_FIXED, fixed=(1.002, 0.3, 0.05, 0.0)),
                      "x+": cases.SideSpec(G_COPY)},
}


@pytest.mark.parametrize("label", ["cavity", "mixed"])
@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_build_rect_case_matches_reference(gold, label, key):
    g = gold(f"ghosts_{label}")
    tag = key.replace(".", "p")
    dp = 1.0 / 20
    spec = kernel_spec(configs.FAMILY[key], 1.3 * dp, 2)
    eos = EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0)
    interior, gpos, gh = cases.build_rect_case((0, 0), (1, 1), dp, spec.kappa * spec.h,
                                               SIDES[label](), eos)
    if label == "mixed":
        bottom = gh.kind == G_MIRROR
        gh.kind[bottom & (gpos[:, 0] > 0.5)] = G_BLEND_MIRROR
    np.testing.assert_array_equal(np.vstack([interior, gpos]), g[f"{tag}__pos"])
    for f in ("kind", "src", "normal", "wall_v", "fixed"):
        np.testing.assert_array_equal(getattr(gh, f), g[f"{tag}__{f}"], err_msg=f)


@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_dmr_frame_matches_reference(gold, key):
    """build_dmr's frame (cases.py:395-416) without constructing the solver."""
    g = gold("hllc_dmr")
    tag = key.replace(".", "p")
    dp = 1.0 / 16
    spec = kernel_spec(configs.FAMILY[key], 1.3 * dp, 2)
    from paper_2405_05155_b200.eulerian import G_DMR_TOP, IDEAL_GAS

    sides = {"x-": cases.SideSpec(G_FIXED, fixed=cases.DMR_POST), "x+": cases.SideSpec(G_COPY),
             "y-": cases.SideSpec(G_MIRROR), "y+": cases.SideSpec(G_DMR_TOP)}
    interior, gpos, gh = cases.build_rect_case(
        (0, 0), (4, 1), dp, spec.kappa * spec.h, sides, EosParams(IDEAL_GAS, gamma=1.4),
        gamma=1.4, dmr_params={"x0": 1.0 / 6.0, "post": cases.DMR_POST, "pre": cases.DMR_PRE})
    np.testing.assert_array_equal(np.vstack([interior, gpos]), g[f"{tag}__pos"])
    np.testing.assert_array_equal(gh.src, g[f"{tag}__src"])
    np.testing.assert_array_equal(gh.fixed, g[f"{tag}__fixed"])
    np.testing.assert_array_equal(gh.dmr["ghost_x"], g[f"{tag}__dmr_ghost_x"])
    np.testing.assert_array_equal(gh.dmr["post"], g[f"{tag}__dmr_post"])
    np.testing.assert_array_equal(gh.dmr["pre"], g[f"{tag}__dmr_pre"])


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_build_dmr_case_vs_reference_golden(gold, key):
    g = gold("hllc_dmr")
    tag = key.replace(".", "p")
    cfg = cases.CaseConfig(name="dmr", case="dmr", solver="euler-hllc", dp=1.0 / 16, t_end=0.2,
                           kernel_family=configs.FAMILY[key])
    case = cases.build_case(cfg)
    s = case.solver
    np.testing.assert_array_equal(s.pos, g[f"{tag}__pos"])
    for f in ("kind", "src", "blend"):
        np.testing.assert_array_equal(getattr(s.ghosts, f), g[f"{tag}__{f}"], err_msg=f)
    st = s.state
    np.testing.assert_array_equal(st.etot, g[f"{tag}__etot_init"])
    for _ in range(20):
        case.advance()
    ni = s.n_int
    assert l2_error(s.state.rho[:ni], g[f"{tag}__rho20"]) < 1e-8
    assert l2_error(s.state.etot[:ni], g[f"{tag}__etot20"]) < 1e-8
    assert case.snapshot_array().shape == (ni, 7)


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_build_cylinder_case_vs_reference_golden(gold, key):
    g = gold("cylinder")
    tag = key.replace(".", "p")
    cfg = cases.CaseConfig(name="cyl", case="cylinder", solver="euler-wc", dp=0.1, t_end=1.0,
                           kernel_family=configs.FAMILY[key],
                           physics={"u_inf": 1.0, "rho0": 1.0, "re": 20.0},
                           geometry={"diameter": 1.0, "extent": (5.0, 3.0),
                                     "center": (1.5, 1.5)})
    s = cases.build_case(cfg).solver
    np.testing.assert_array_equal(s.pos, g[f"{tag}__pos"])
    for f in ("kind", "src", "wall_v", "fixed"):
        np.testing.assert_array_equal(getattr(s.ghosts, f), g[f"{tag}__{f}"], err_msg=f)
    np.testing.assert_allclose(s.ghosts.normal, g[f"{tag}__normal"], rtol=0, atol=1e-12)
    for _ in range(30):
        s.step()
    assert l2_error(s.state.rho[:s.n_int], g[f"{tag}__rho30"]) < 1e-8
    wf = np.array([w for _, w in s.wall_force_series])
    assert l2_error(wf, g[f"{tag}__wf"]) < 1e-8


@pytest.mark.gpu
def test_other_builders_run():
    """Cavity, shear layer, twist / bend columns and the semicircular cavity
    (GPU relaxation inside a half disk) build and step."""
    for case, extra in (("cavity", {"physics": {"re": 100.0}}), ("shear-layer", {}),
                        ("semicircle-cavity", {"relax": {"max_steps": 20}})):
        cfg = cases.CaseConfig(name=case, case=case, solver="euler-wc", dp=0.05, t_end=0.1,
                               **extra)
        c = cases.build_case(cfg)
        for _ in range(3):
            c.advance()
        assert np.isfinite(c.snapshot_array()).all()
    for case in ("twist", "bend"):
        cfg = cases.CaseConfig(name=case, case=case, solver="tlsph", dp=0.25, t_end=0.1,
                               h_ratio=1.15, cfl=0.6)
        c = cases.build_case(cfg)
        for _ in range(3):
            c.advance()
        c.record_outputs()
        assert np.isfinite(c.snapshot_array()).all() and c.vm_max > 0.0


def test_load_config(tmp_path):
    """TOML case files: defaults, tables passed through, and the checks of
    cases.py:82-118 (unknown case / family, dp, t_end)."""
    from paper_2405_05155_b200.eulerian import ConfigError

    f = tmp_path / "cav.toml"
    f.write_text('case = "cavity"\ndp = 0.05\nt_end = 1.0\n[kernel]\nfamily = "wendland-truncated"\n'
                 'h_ratio = 1.3\n[physics]\nre = 400.0\nu_wall = 1.0\n[output]\nevery = 0.5\n')
    cfg = cases.load_config(f)
    assert (cfg.name, cfg.case, cfg.dp, cfg.t_end) == ("cav", "cavity", 0.05, 1.0)
    assert (cfg.kernel_family, cfg.h_ratio, cfg.cfl, cfg.correction) == \
        ("wendland-truncated", 1.3, 0.5, True)
    assert cfg.physics == {"re": 400.0, "u_wall": 1.0} and cfg.output_every == 0.5
    assert cfg.kernel(2).kappa == 1.6
    relax = tmp_path / "r.toml"
    relax.write_text('case = "relax"\ndp = 0.1\n[geometry]\nkind = "semicircle"\nradius = 0.5\n')
    rc = cases.load_config(relax)
    assert isinstance(cases._shape_from_geometry(rc.geometry), cases.geometry.SemiCircle)
    for body in ('case = "nope"\ndp = 0.1\nt_end = 1.0\n', 'case = "cavity"\nt_end = 1.0\n',
                 'case = "cavity"\ndp = -1.0\nt_end = 1.0\n', 'case = "cavity"\ndp = 0.1\n',
                 'case = "cavity"\ndp = 0.1\nt_end = 1.0\n[kernel]\nfamily = "gauss"\n'):
        bad = tmp_path / "bad.toml"
        bad.write_text(body)
        with pytest.raises(ConfigError):
            cases.load_config(bad)
    with pytest.raises(ConfigError):
        cases.load_config(tmp_path / "missing.toml")
    with pytest.raises(ConfigError):
        cases._shape_from_geometry({"kind": "torus"})
