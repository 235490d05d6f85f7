"""API surface around the hot path against fixtures written by the reference
itself (tests/golden/surface.npz, make_golden.py section "surface"):
pairwise Riemann helpers (eulerian.py:90-219), dmr_shock_x and the
module-level apply_boundaries (:366-447), EulerianSolver.viscous_rhs
(:645-653)."""

import numpy as np
import pytest

from paper_2405_05155_b200 import cases, configs, eulerian
from paper_2405_05155_b200.eulerian import (G_BLEND_MIRROR, G_COPY, G_FIXED, G_MIRROR, G_WALL,
                                            WEAKLY_COMPRESSIBLE, EosParams, FluidState,
                                            InterfaceState)
from paper_2405_05155_b200.kernels import kernel_spec


def _states(g, k):
    a = g[f"state{k}"]
    d = a.shape[1] - 4
    return [InterfaceState(rho=r[0], v=tuple(r[4:4 + d]), p=r[1], c=r[2], etot=r[3]) for r in a]


@pytest.mark.parametrize("which", ["linearized", "hllc"])
def test_riemann_helpers_match_reference(gold, which):
    g = gold("surface")
    fn = eulerian.linearized_star if which == "linearized" else eulerian.hllc_star
    for k in range(40):
        left, right = _states(g, k)
        r = fn(left, right, g[f"e{k}"])
        d = len(left.v)
        got = [r.u_star, r.p_star, r.rho_star_l, r.rho_star_r, r.e_star_l, r.e_star_r, r.s_l,
               r.s_r, r.s_star, r.beta] + list(r.v_star) + [0.0] * (3 - d)
        np.testing.assert_allclose(got, g[which][k], rtol=1e-15, atol=1e-15)


def test_dmr_shock_x_matches_reference(gold):
    g = gold("surface")
    np.testing.assert_array_equal([eulerian.dmr_shock_x(t) for t in (0.0, 0.05, 0.2)], g["dmr_x"])


def test_module_apply_boundaries_wc_matches_reference(gold):
    g = gold("surface")
    dp = 1.0 / 20
    spec = kernel_spec("wendland-truncated", 1.3 * dp, 2)
    eos = EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0)
    interior, gpos, ghosts = cases.build_rect_case(
        (0, 0), (1, 1), dp, spec.kappa * spec.h,
        {"y+": cases.SideSpec(G_WALL, wall_v=(0.5, 0.0)), "y-": cases.SideSpec(G_MIRROR),
         "x-": cases.SideSpec(G_FIXED, fixed=(1.002, 0.3, 0.05, 0.0)),
         "x+": cases.SideSpec(G_COPY)}, eos)
    bottom = ghosts.kind == G_MIRROR
    ghosts.kind[bottom & (gpos[:, 0] > 0.5)] = G_BLEND_MIRROR
    ghosts.blend = np.clip(gpos[:, 0] - 0.4, 0.0, 1.0)
    n = interior.shape[0] + gpos.shape[0]
    st = FluidState(vol=np.full(n, dp * dp), rho=g["wc_rho_in"].copy(),
                    mom=g["wc_mom_in"].copy(), etot=None, n_interior=interior.shape[0])
    eulerian.apply_boundaries(st, ghosts, eos, 0.0)
    np.testing.assert_allclose(st.rho, g["wc_rho_out"], rtol=1e-15, atol=0)
    np.testing.assert_allclose(st.mom, g["wc_mom_out"], rtol=1e-14, atol=1e-16)


def test_module_apply_boundaries_dmr_matches_reference(gold):
    """Ideal gas, fixed / copy / blend-mirror / moving-shock ghosts."""
    g = gold("surface")
    dp = 1.0 / 16
    spec = kernel_spec("wendland-truncated", 1.3 * dp, 2)
    eos = eulerian.EosParams(eulerian.IDEAL_GAS, gamma=1.4)
    sides = {"x-": cases.SideSpec(G_FIXED, fixed=cases.DMR_POST), "x+": cases.SideSpec(G_COPY),
             "y-": cases.SideSpec(G_MIRROR), "y+": cases.SideSpec(eulerian.G_DMR_TOP)}
    interior, gpos, ghosts = cases.build_rect_case(
        (0, 0), (4, 1), dp, spec.kappa * spec.h, sides, eos, gamma=1.4,
        dmr_params={"x0": 1.0 / 6.0, "post": cases.DMR_POST, "pre": cases.DMR_PRE})
    floor = (ghosts.kind == G_MIRROR) & (gpos[:, 1] < 0.0)
    ghosts.kind[floor] = G_BLEND_MIRROR
    ghosts.blend = np.where(floor, np.clip((gpos[:, 0] - 1.0 / 6.0) / (spec.kappa * spec.h),
                                           0.0, 1.0), 0.0)
    n = interior.shape[0] + gpos.shape[0]
    st = FluidState(vol=np.full(n, dp * dp), rho=g["dmr_rho_in"].copy(),
                    mom=g["dmr_mom_in"].copy(), etot=g["dmr_etot_in"].copy(),
                    n_interior=interior.shape[0])
    eulerian.apply_boundaries(st, ghosts, eos, 0.07)
    np.testing.assert_allclose(st.rho, g["dmr_rho_out"], rtol=1e-15, atol=0)
    np.testing.assert_allclose(st.mom, g["dmr_mom_out"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(st.etot, g["dmr_etot_out"], rtol=1e-14, atol=1e-14)


@pytest.mark.gpu
def test_viscous_rhs_matches_reference(gold):
    from paper_2405_05155_b200.approx import l2_error

    g = gold("surface")
    cfg = configs.c2_tgv2d(kernel="1.6h", n_side=32)
    n = cfg["pos"].shape[0]
    s = eulerian.EulerianSolver(cfg["pos"], n, FluidState(cfg["vol"].copy(), cfg["rho"].copy(),
                                                          cfg["mom"].copy(), None, n),
                                EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0),
                                cfg["spec"], None, cfl=cfg["cfl"], mu=cfg["mu"],
                                periodic_box=cfg["box"])
    assert l2_error(s.viscous_rhs(), g["viscous_rhs"]) < 1e-13
