"""Command line (paper_2405_05155_b200/cli.py; reference cli.py): parser,
exit codes, and — on a GPU — each sub-command end to end on tiny inputs."""

import json

import numpy as np
import pytest

from paper_2405_05155_b200 import cli, harness


def test_parser_and_config_errors(tmp_path, capsys):
    args = cli.build_parser().parse_args(["run", "case.toml", "--out", "o", "--seed", "3"])
    assert (args.command, args.config, args.out, args.seed) == ("run", "case.toml", "o", 3)
    assert cli.main(["run", str(tmp_path / "missing.toml")]) == 3
    bad = tmp_path / "bad.toml"
    bad.write_text('case = "warp-drive"\ndp = 0.1\nt_end = 1.0\n')
    assert cli.main(["pair", str(bad)]) == 3
    assert "config error" in capsys.readouterr().err


def test_reference_profile_tables(tmp_path):
    """load_reference_profile / compare_profiles on a table in the Ghia
    file format (comments, header, coordinate,value rows)."""
    tab = tmp_path / "profile.csv"
    tab.write_text("# synthetic table\ny,u\n0.0,0.0\n0.5,-0.2\n1.0,1.0\n")
    y, u = harness.load_reference_profile(str(tab))
    np.testing.assert_array_equal(y, [0.0, 0.5, 1.0])
    np.testing.assert_array_equal(u, [0.0, -0.2, 1.0])
    m = harness.compare_profiles(y, u + np.array([0.3, 0.1, -0.3]), y, u, skip_boundary=(0.0, 1.0))
    assert m["l2"] == pytest.approx(0.1) and m["linf"] == pytest.approx(0.1)
    y2, _ = harness.load_reference_profile("profile.csv", data_dir=tmp_path)
    np.testing.assert_array_equal(y, y2)
    from paper_2405_05155_b200.eulerian import ConfigError

    with pytest.raises(ConfigError):
        harness.load_reference_profile("nope.csv", data_dir=tmp_path)


@pytest.mark.gpu
def test_cli_commands_on_gpu(tmp_path, capsys):
    cav = tmp_path / "cav.toml"
    cav.write_text('case = "cavity"\ndp = 0.1\nt_end = 0.02\n[physics]\nre = 100.0\n')
    assert cli.main(["run", str(cav), "--out", str(tmp_path / "run")]) == 0
    rep = json.loads((tmp_path / "run" / "cav-report.json").read_text())
    assert rep["steps"] > 0 and np.isfinite(rep["conservation"]["mass_rel_drift"])
    assert cli.main(["pair", str(cav), "--out", str(tmp_path / "pair")]) == 0
    assert "alpha" in capsys.readouterr().out
    rel = tmp_path / "relax.toml"
    rel.write_text('case = "relax"\ndp = 0.2\n[geometry]\nkind = "circle"\ndiameter = 2.0\n'
                   '[relax]\nmax_steps = 10\n')
    assert cli.main(["relax", str(rel), "--out", str(tmp_path / "rel")]) == 0
    pos = np.loadtxt(tmp_path / "rel" / "relax-positions.csv", delimiter=",", skiprows=1)
    assert pos.shape[1] == 3 and np.all(np.hypot(pos[:, 0], pos[:, 1]) < 1.0)
    study = tmp_path / "study.toml"
    study.write_text('[study]\nresolutions = [0.2, 0.1]\ndistributions = ["lattice"]\n')
    assert cli.main(["error-study", str(study), "--out", str(tmp_path / "es")]) == 0
    rows = (tmp_path / "es" / "error-study.csv").read_text().splitlines()
    assert len(rows) == 1 + 2 * 2 * 2
