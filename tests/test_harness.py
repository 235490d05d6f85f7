"""Harness: paired standard/truncated runs, reports,
snapshots and the drag/lift reduction against the reference's own harness
(tests/golden/harness.npz from sph_trunc.bench)."""

import json

import numpy as np
import pytest

from paper_2405_05155_b200 import harness
from paper_2405_05155_b200.cases import CaseConfig


def test_drag_lift_matches_reference(gold):
    g = gold("harness")
    dl = harness.drag_lift(g["drag__t"], g["drag__f"], 1.0, 1.0, 2.0)
    np.testing.assert_array_equal(dl["cd"], g["drag__cd"])
    np.testing.assert_array_equal(dl["cl"], g["drag__cl"])
    np.testing.assert_allclose([dl["strouhal"], dl["cd_mean_tail"], dl["cl_amplitude_tail"]],
                               g["drag__scalars"], rtol=1e-14)
    with pytest.raises(ValueError):
        harness.drag_lift([0.0], [1.0], 1.0, 1.0, 1.0)
    assert harness.alpha_ratio(1.0, 2.0) == 0.5
    with pytest.raises(ValueError):
        harness.alpha_ratio(0.0, 1.0)


@pytest.mark.gpu
def test_paired_shear_layer_matches_reference(gold, tmp_path):
    """Shear layer, standard then truncated Wendland: steps, dt range,
    neighbour statistics, conservation, alpha and the field differences."""
    g = gold("harness")
    cfg = CaseConfig(name="shear", case="shear-layer", solver="euler-wc", dp=1.0 / 32,
                     t_end=0.04, kernel_family="wendland", h_ratio=1.3, cfl=0.5,
                     output_every=0.02)
    pair, case_sw, case_tw = harness.paired_run(cfg, out_dir=tmp_path)
    for leg, rep in (("sw", pair.sw), ("tw", pair.tw)):
        assert rep.steps == int(g[f"shear_{leg}__steps"])
        assert rep.t_end == pytest.approx(float(g[f"shear_{leg}__t_end"]), rel=1e-12)
        ns = [rep.neighbor_stats[k] for k in ("mean", "min", "max", "pairs")]
        np.testing.assert_allclose(ns, g[f"shear_{leg}__nstats"], rtol=0)
        assert rep.conservation["mass_rel_drift"] < 1e-13
        np.testing.assert_allclose([rep.diagnostics["dt_min"], rep.diagnostics["dt_max"]],
                                   g[f"shear_{leg}__dt"], rtol=1e-10)
    assert pair.alpha > 0.0
    assert pair.field_diff["velocity_l2"] == pytest.approx(float(g["shear__velocity_l2"]),
                                                           rel=1e-6)
    assert pair.field_diff["vorticity_l2"] == pytest.approx(float(g["shear__vorticity_l2"]),
                                                            rel=1e-6)
    w = harness.vorticity(case_tw)
    assert np.linalg.norm(w - g["shear_tw__vorticity"]) / np.linalg.norm(
        g["shear_tw__vorticity"]) < 1e-8
    rep = json.loads((tmp_path / "shear-pair.json").read_text())
    assert rep["alpha"] == pytest.approx(pair.alpha)
    snap = np.loadtxt(tmp_path / "shear-tw-final.csv", delimiter=",", skiprows=1)
    assert snap.shape == (1024, 6)
    assert (tmp_path / "shear-sw-0001.csv").exists()


@pytest.mark.gpu
def test_run_case_solid_column(tmp_path):
    cfg = CaseConfig(name="bend", case="bend", solver="tlsph", dp=0.25, t_end=2e-4,
                     h_ratio=1.15, cfl=0.6, output_every=1e-4)
    rep, case = harness.run_case(cfg, out_dir=tmp_path)
    assert rep.steps > 0 and rep.t_end == pytest.approx(2e-4)
    assert rep.metrics["von_mises_max"] > 0.0
    assert (tmp_path / "bend-tip.csv").exists() and (tmp_path / "bend-report.json").exists()
