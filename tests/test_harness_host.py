"""Artifact writers and run configuration (no GPU).

The reference's ``run_single`` artifacts (`harness/experiments.py:102-117`,
`harness/reports.py:24-63`, `grid.py:100-110`) were captured from the
unmodified reference (``make_golden.py harness``).  Rebuilding a report from
the captured report.json and writing it with this package's writers must give
byte-identical files: same JSON layout, same float spelling, same CSV rows.
"""

import json

import numpy as np
import pytest

from conftest import golden
from paper_2411_00546_b200.grid import Grid
from paper_2411_00546_b200.harness import (ConfigError, ExperimentConfig, config_to_dict,
                                           read_field_csv, report_to_dict, sparsity_fraction,
                                           write_field_csv, write_report_json,
                                           write_residual_history_csv)
from paper_2411_00546_b200.newton import SolveReport

CASES = ["newton_eps", "newton", "newton_eps_gmres", "newton_ras_eps", "raspen_eps",
         "raspen_eps_23", "fail_max_outer"]


def _report_from(d):
    return SolveReport(converged=d["converged"], outer_iters=d["outer_iters"],
                       residual_norms=d["residual_history"], eps_values=d["eps_history"],
                       alphas=d["alphas"], gmres_iters=d["gmres_iters"],
                       inner_iters=d["inner_iters"], threshold=d["threshold"],
                       wall_time=d["timing"]["wall_time_s"], failure=d["failure"])


@pytest.mark.parametrize("tag", CASES)
def test_writers_reproduce_reference_artifacts_bytewise(tag, tmp_path):
    g = golden("harness.npz")
    ref_json = str(g[f"{tag}__report.json"])
    d = json.loads(ref_json)
    cfg = ExperimentConfig(**d["config"])
    assert config_to_dict(cfg) == d["config"]
    rep = _report_from(d)
    assert rep.avg_gmres_iters == d["avg_gmres_iters"]
    assert rep.avg_inner_iters == d["avg_inner_iters"]
    grid = Grid(cfg.n)
    ref_u = str(g[f"{tag}__u.csv"])
    (tmp_path / "ref_u.csv").write_text(ref_u)
    u = read_field_csv(tmp_path / "ref_u.csv", grid)
    data = report_to_dict(config_to_dict(cfg), rep, sparsity_fraction=sparsity_fraction(u))
    write_report_json(tmp_path / "report.json", data)
    assert (tmp_path / "report.json").read_text() == ref_json
    write_residual_history_csv(tmp_path / "residual_history.csv", rep)
    assert (tmp_path / "residual_history.csv").read_text() == str(g[f"{tag}__residual_history.csv"])
    for name in ("y.csv", "p.csv", "u.csv"):
        (tmp_path / f"ref_{name}").write_text(str(g[f"{tag}__{name}"]))
        v = read_field_csv(tmp_path / f"ref_{name}", grid)
        write_field_csv(tmp_path / name, grid, v)
        assert (tmp_path / name).read_text() == str(g[f"{tag}__{name}"])


def test_config_validation_mirrors_reference():
    with pytest.raises(ConfigError, match="unknown method"):
        ExperimentConfig(method="bogus")
    with pytest.raises(ConfigError, match="direct linear solver is incompatible"):
        ExperimentConfig(method="newton-ras-eps", linear_solver="direct")
    with pytest.raises(ConfigError, match="matrix-free"):
        ExperimentConfig(method="raspen", linear_solver="direct")
    with pytest.raises(ConfigError, match="eps0 >= eps_min"):
        ExperimentConfig(eps0=1e-12)
    cfg = ExperimentConfig()
    assert cfg.method == "newton-eps" and cfg.subdomains == "1x1" and cfg.uses_continuation


def test_sparsity_fraction():
    assert sparsity_fraction(np.zeros(4)) == 1.0
    assert sparsity_fraction(np.array([1.0, 1e-9, 0.0, -2.0])) == 0.5
