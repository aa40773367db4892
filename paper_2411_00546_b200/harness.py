"""Single-run orchestration and artifacts for GPU runs.

Mirror of the reference's `harness/config.py` (the ``ExperimentConfig`` fields,
defaults and validation), `harness/experiments.py:35-117` (``build_problem``,
``schedule_for``, ``solve_single``, ``run_single``, ``sparsity_fraction``) and
`harness/reports.py:1-63` + `grid.py:100-110` (report.json, residual history
CSV and field CSVs, same formats: JSON with sorted keys and indent 2, floats by
repr, fields by ``%.17g``).  Every method runs on the device:

* ``raspen`` / ``raspen-eps``      -> ``schwarz.raspen_solve``
* ``newton-ras`` / ``newton-ras-eps`` -> ``linear_ras.newton_ras_solve``
* ``newton`` / ``newton-eps``      -> monolithic Newton on the global residual;
  ``linear_solver`` auto/direct: one block-Thomas factorisation of the whole Jacobian
  (single-subdomain engine, block factor of the whole grid), gmres: unpreconditioned
  device GMRES.

The manufactured problem of ``build_problem`` is set up on the device
(``problem_setup.construct_test_problem``).
"""

import csv
import json
from dataclasses import dataclass, fields, replace
from pathlib import Path

import numpy as np

from .grid import Grid
from .krylov import KrylovConfig
from .linear_ras import GlobalJacobian, global_residual, newton_ras_solve
from .newton import ContinuationSchedule, NewtonConfig, newton_continuation
from .problem_setup import construct_test_problem, grid_engine
from .schwarz import build_local_systems, decompose, raspen_solve
from .system import recover_control, split_pair

METHODS = ("newton", "newton-eps", "newton-ras", "newton-ras-eps", "raspen", "raspen-eps")
LINEAR_SOLVERS = ("auto", "direct", "gmres")
SCHEMA_VERSION = 1
SPARSITY_THRESHOLD = 1e-8


class ConfigError(ValueError):
    """Invalid experiment configuration (`harness/config.py:15-16`)."""


@dataclass(frozen=True)
class ExperimentConfig:
    """`harness/config.py:19-90`: same fields, defaults and checks."""

    method: str = "newton-eps"
    n: int = 64
    s1: int = 1
    s2: int = 1
    overlap: int = 2
    eps0: float = 1.0
    gamma: float = 0.2
    eps_min: float = 1e-10
    tol: float = 1e-10
    sigma: float = 1.1
    inner_tol: float = 1e-8
    kappa: float = 0.1
    nu: float = 1e-6
    mu: float = 1.0
    k_tilde: int = 5
    seed: int = 0
    threads: int = 1
    linear_solver: str = "auto"
    gmres_tol: float = 1e-8
    max_outer: int = 200

    def __post_init__(self):
        if self.method not in METHODS:
            raise ConfigError(f"unknown method {self.method!r}; choose from {', '.join(METHODS)}")
        if self.linear_solver not in LINEAR_SOLVERS:
            raise ConfigError(f"unknown linear solver {self.linear_solver!r}")
        if self.n < 1:
            raise ConfigError("n must be at least 1")
        if self.s1 < 1 or self.s2 < 1:
            raise ConfigError("subdomain counts must be at least 1")
        if self.overlap < 0:
            raise ConfigError("overlap must be nonnegative")
        if not self.eps0 >= self.eps_min > 0:
            raise ConfigError("need eps0 >= eps_min > 0")
        if not 0.0 < self.gamma <= 1.0:
            raise ConfigError("gamma must lie in (0, 1]")
        if self.tol <= 0 or self.inner_tol <= 0:
            raise ConfigError("tolerances must be positive")
        if self.sigma < 1.0:
            raise ConfigError("sigma must be at least 1")
        if self.nu <= 0 or self.mu <= 0:
            raise ConfigError("nu and mu must be positive")
        if self.threads < 0:
            raise ConfigError("threads must be nonnegative")
        if self.max_outer < 0:
            raise ConfigError("max_outer must be nonnegative")
        if self.uses_ras and self.linear_solver == "direct":
            raise ConfigError(f"method {self.method} preconditions GMRES; "
                              "a direct linear solver is incompatible")
        if self.is_raspen and self.linear_solver == "direct":
            raise ConfigError("raspen solves its outer system matrix-free; "
                              "a direct linear solver is incompatible")

    @property
    def uses_ras(self):
        return self.method in ("newton-ras", "newton-ras-eps")

    @property
    def is_raspen(self):
        return self.method in ("raspen", "raspen-eps")

    @property
    def uses_continuation(self):
        return self.method.endswith("-eps")

    @property
    def subdomains(self):
        return f"{self.s1}x{self.s2}"


def config_to_dict(cfg):
    return {f.name: getattr(cfg, f.name) for f in fields(cfg)}


def with_updates(cfg, **kwargs):
    return replace(cfg, **kwargs)


def build_problem(cfg):
    grid = Grid(cfg.n)
    spec, _ = construct_test_problem(grid, kappa=cfg.kappa, nu=cfg.nu, mu=cfg.mu,
                                     k_tilde=cfg.k_tilde)
    return grid, spec


def schedule_for(cfg):
    """Continuation methods walk eps0 -> eps_min; plain ones sit at eps_min."""
    if cfg.uses_continuation:
        return ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)
    return ContinuationSchedule.fixed(cfg.eps_min)


def _monolithic(cfg, spec, sched, x0):
    """`experiments.py:86-91` on the device: direct solves on a single-subdomain
    engine (one block-Thomas factorisation of the whole Jacobian), GMRES on a grid-only one."""
    if cfg.linear_solver in ("auto", "direct"):
        lin = "direct"
        engine = build_local_systems(decompose(spec.grid, 1, 1, 0), spec)
    else:
        lin = KrylovConfig(rel_tol=cfg.gmres_tol, max_iters=5000)
        engine = grid_engine(spec)
    newton_cfg = NewtonConfig(tol=cfg.tol, max_outer=cfg.max_outer, sigma=cfg.sigma,
                              linear_solver=lin)
    x, report = newton_continuation(
        engine.from_host(x0), lambda x, eps: global_residual(engine, x, eps),
        lambda x, eps: GlobalJacobian(engine, x, eps), sched, newton_cfg)
    return x.to_host(), report


def solve_single(cfg, spec=None):
    """Dispatch one solve per the configured method; returns (x, report, spec)."""
    if spec is None:
        _, spec = build_problem(cfg)
    sched = schedule_for(cfg)
    x0 = np.zeros(2 * spec.grid.size)
    if cfg.is_raspen:
        dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
        x, report = raspen_solve(
            x0, dec, spec, sched,
            cfg=NewtonConfig(tol=cfg.tol, max_outer=cfg.max_outer, sigma=cfg.sigma),
            krylov_cfg=KrylovConfig(rel_tol=cfg.gmres_tol, max_iters=1000),
            inner_tol=cfg.inner_tol, threads=cfg.threads,
            continuation=cfg.uses_continuation)
        return x, report, spec
    if cfg.uses_ras:
        dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
        newton_cfg = NewtonConfig(tol=cfg.tol, max_outer=cfg.max_outer, sigma=cfg.sigma,
                                  linear_solver=KrylovConfig(rel_tol=cfg.gmres_tol,
                                                             max_iters=2000))
        x, report = newton_ras_solve(x0, dec, spec, sched, newton_cfg)
        return x, report, spec
    x, report = _monolithic(cfg, spec, sched, x0)
    return x, report, spec


def sparsity_fraction(u, threshold=SPARSITY_THRESHOLD):
    """Share of entries below threshold * ||u||_inf (1.0 for the zero field)."""
    scale = np.abs(u).max()
    if scale == 0.0:
        return 1.0
    return float(np.mean(np.abs(u) < threshold * scale))


# ---------------------------------------------------------------------------
# artifacts (`harness/reports.py:1-63`, `grid.py:100-110`)
# ---------------------------------------------------------------------------

def _fmt(value):
    if value is None:
        return ""
    if isinstance(value, float):
        return repr(value)
    return str(value)


def report_to_dict(cfg_dict, report, sparsity_fraction=None):
    avg_g = report.avg_gmres_iters
    avg_i = report.avg_inner_iters
    data = {
        "schema": SCHEMA_VERSION,
        "config": dict(cfg_dict),
        "converged": bool(report.converged),
        "outer_iters": int(report.outer_iters),
        "threshold": float(report.threshold),
        "eps_history": [float(e) for e in report.eps_values],
        "residual_history": [float(r) for r in report.residual_norms],
        "alphas": [float(a) for a in report.alphas],
        "gmres_iters": [None if k is None else int(k) for k in report.gmres_iters],
        "inner_iters": [int(k) for k in report.inner_iters],
        "avg_gmres_iters": avg_g,
        "avg_inner_iters": avg_i,
        "failure": report.failure,
        "timing": {"wall_time_s": float(report.wall_time)},
    }
    if sparsity_fraction is not None:
        data["sparsity_fraction"] = float(sparsity_fraction)
    return data


def write_report_json(path, data):
    Path(path).write_text(json.dumps(data, indent=2, sort_keys=True) + "\n", encoding="utf-8")


def read_report_json(path):
    return json.loads(Path(path).read_text(encoding="utf-8"))


def write_residual_history_csv(path, report):
    """One row per outer iterate; iterate 0 has no step, so alpha/gmres are empty."""
    with open(path, "w", newline="", encoding="utf-8") as fh:
        writer = csv.writer(fh)
        writer.writerow(["iteration", "eps", "residual", "alpha", "gmres_iters"])
        for k, (eps, res) in enumerate(zip(report.eps_values, report.residual_norms)):
            alpha = report.alphas[k - 1] if 1 <= k <= len(report.alphas) else None
            gm = report.gmres_iters[k - 1] if 1 <= k <= len(report.gmres_iters) else None
            writer.writerow([k, _fmt(eps), _fmt(res), _fmt(alpha), _fmt(gm)])


def write_field_csv(path, grid, v):
    """One CSV row per grid row, row-major, full precision (`grid.py:100-102`)."""
    np.savetxt(path, np.asarray(v).reshape(grid.n, grid.n), delimiter=",", fmt="%.17g")


def read_field_csv(path, grid):
    vals = np.loadtxt(path, delimiter=",", ndmin=2)
    if vals.shape != (grid.n, grid.n):
        raise ValueError(f"field file {path} has shape {vals.shape}, expected {(grid.n, grid.n)}")
    return vals.ravel()


def run_single(cfg, out_dir, spec=None):
    """One configured solve plus its artifact set; returns (exit_code, report dict)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    x, report, spec = solve_single(cfg, spec)
    y, p = split_pair(x)
    u = recover_control(p, spec, cfg.eps_min)
    data = report_to_dict(config_to_dict(cfg), report, sparsity_fraction=sparsity_fraction(u))
    write_report_json(out / "report.json", data)
    write_residual_history_csv(out / "residual_history.csv", report)
    write_field_csv(out / "y.csv", spec.grid, y)
    write_field_csv(out / "p.csv", spec.grid, p)
    write_field_csv(out / "u.csv", spec.grid, u)
    return (0 if report.converged else 3), data
