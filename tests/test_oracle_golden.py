"""Pin the CPU oracle to fixtures produced by the UNMODIFIED reference.

The fixtures come from ``tests/golden/make_golden.py`` (reference imported
from /root/reference/pkg/src in the build container).  The oracle restates
the reference's algorithm with the same library calls, so it must agree
bitwise on everything it recomputes here.
"""

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

import raspen_oracle as O
from conftest import golden
from paper_2411_00546_b200.problems import CONFIGS, build_fields, mild_spec
from paper_2411_00546_b200.system import Nonlinearity, make_phi

UNIT_CASES = [
    ("kappa16", 16, 2, 2, 2, Nonlinearity(0.1), 1e-2, 1.0),
    ("cubic20", 20, 2, 3, 2, make_phi("cubic"), 1e-3, 1e-2),
    ("expm1_18", 18, 3, 2, 3, make_phi("expm1"), 1e-4, 5e-3),
]


def unit_problem(n, s1, s2, m, phi, nu, mu):
    base = mild_spec(n)
    return O.Problem(n, s1, s2, m, phi, nu, mu, base.f, 10.0 * base.y_d)


@pytest.mark.parametrize("case", UNIT_CASES, ids=[c[0] for c in UNIT_CASES])
def test_oracle_units_bitwise(case):
    tag, n, s1, s2, m, phi, nu, mu = case
    g = golden("units.npz")
    prob = unit_problem(n, s1, s2, m, phi, nu, mu)
    x = g[f"{tag}_x"]
    eps = 1e-2
    loc = np.concatenate([prob.local_fns(i, x)[0](x[r.pair_idx] + 0.01, eps)
                          for i, r in enumerate(prob.rects)])
    np.testing.assert_array_equal(loc, g[f"{tag}_local_res"])
    f_val, corr = O.raspen_residual(prob, x, eps, tol=1e-10, threads=1)
    np.testing.assert_array_equal(f_val, g[f"{tag}_fval"])
    assert corr.inner == list(g[f"{tag}_inner"])
    out = O.raspen_jvp(prob, x, g[f"{tag}_d"], eps, corr)
    np.testing.assert_array_equal(out, g[f"{tag}_jvp"])
    xs, rep = O.raspen_solve(prob, np.zeros_like(x), 1.0, 0.2, 1e-3, threads=1)
    np.testing.assert_array_equal(xs, g[f"{tag}_solve_x"])
    assert rep["outer_iters"] == int(g[f"{tag}_solve_outer"])
    assert rep["inner_iters"] == list(g[f"{tag}_solve_inner"])
    assert rep["gmres_iters"] == list(g[f"{tag}_solve_gmres"])
    assert rep["per_sub"] == g[f"{tag}_solve_per_sub"].tolist()


def _cfg_problem(name):
    cfg = CONFIGS[name]
    f, yd = build_fields(cfg)
    return cfg, O.Problem(cfg.n, cfg.s1, cfg.s2, cfg.overlap, make_phi(cfg.phi), cfg.nu,
                          cfg.mu, f, yd)


def test_oracle_cfg1_bitwise():
    g = golden("cfg1_tol1e-08.npz")
    cfg, prob = _cfg_problem("cfg1")
    x, rep = O.raspen_solve(prob, np.zeros(cfg.unknowns), cfg.eps0, cfg.gamma, cfg.eps_min,
                            threads=1)
    n2 = cfg.n * cfg.n
    np.testing.assert_array_equal(x[:n2], g["y"])
    np.testing.assert_array_equal(x[n2:], g["p"])
    assert rep["outer_iters"] == int(g["outer_iters"]) == 3
    assert rep["inner_iters"] == list(g["inner_iters"]) == [7, 2, 1, 1]
    assert rep["gmres_iters"] == list(g["gmres_iters"]) == [13, 14, 14]
    assert rep["per_sub"] == g["per_sub"].tolist()
    np.testing.assert_array_equal(rep["residual_norms"], g["residual_norms"])
    u = O.recover_control(x[n2:], cfg.mu, cfg.nu, cfg.eps_min)
    np.testing.assert_array_equal(u, g["u"])


@pytest.mark.slow
def test_oracle_cfg2_bitwise():
    g = golden("cfg2_tol1e-08.npz")
    cfg, prob = _cfg_problem("cfg2")
    # the fixture was made with single-threaded BLAS (dot order depends on it)
    with threadpool_limits(1, user_api="blas"):
        x, rep = O.raspen_solve(prob, np.zeros(cfg.unknowns), cfg.eps0, cfg.gamma, cfg.eps_min)
    n2 = cfg.n * cfg.n
    np.testing.assert_array_equal(x[:n2], g["y"])
    np.testing.assert_array_equal(x[n2:], g["p"])
    assert rep["inner_iters"] == list(g["inner_iters"])
    assert rep["gmres_iters"] == list(g["gmres_iters"])
    assert rep["per_sub"] == g["per_sub"].tolist()


def test_golden_records_are_consistent():
    """Each golden solve record satisfies its own invariants (len(inner) = outer + 1 etc.)."""
    import glob
    import os
    from conftest import GOLDEN
    for path in sorted(glob.glob(os.path.join(GOLDEN, "cfg[1-4]_tol*.npz"))):
        g = np.load(path)
        if bool(g["converged"]):
            assert len(g["inner_iters"]) == int(g["outer_iters"]) + 1, path
            assert len(g["gmres_iters"]) == int(g["outer_iters"]), path
            assert g["residual_norms"][-1] <= g["threshold"], path
            assert g["per_sub"].shape[0] == len(g["inner_iters"]), path
            np.testing.assert_array_equal(g["per_sub"].max(axis=1), g["inner_iters"])
        else:
            assert "subdomain" in str(g["failure"]), path


# ---------------------------------------------------------------------------
# linear-RAS Newton-Krylov (newton-ras-eps): global residual / Jacobian, the
# RAS preconditioner and full solves, fixtures from the unmodified reference
# (make_golden.py ras_units / ras_cfg1 / ras_cfg2)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("case", UNIT_CASES, ids=[c[0] for c in UNIT_CASES])
def test_oracle_ras_units_bitwise(case):
    tag, n, s1, s2, m, phi, nu, mu = case
    g = golden("ras_units.npz")
    prob = unit_problem(n, s1, s2, m, phi, nu, mu)
    x, d, eps = g[f"{tag}_x"], g[f"{tag}_d"], 1e-2
    np.testing.assert_array_equal(O.global_residual(prob, x, eps), g[f"{tag}_resid"])
    np.testing.assert_array_equal(O.global_jacobian(prob, x, eps) @ d, g[f"{tag}_jvp"])
    np.testing.assert_array_equal(O.ras_preconditioner(prob, x, eps)(d), g[f"{tag}_prec"])
    with threadpool_limits(1, "blas"):
        xs, rep = O.newton_ras_solve(prob, np.zeros_like(x), 1.0, 0.2, 1e-3)
    np.testing.assert_array_equal(xs, g[f"{tag}_solve_x"])
    assert rep["outer_iters"] == int(g[f"{tag}_solve_outer"])
    assert rep["gmres_iters"] == list(g[f"{tag}_solve_gmres"])
    assert rep["alphas"] == list(g[f"{tag}_solve_alphas"])
    np.testing.assert_array_equal(rep["residual_norms"], g[f"{tag}_solve_norms"])


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_oracle_ras_cfg_bitwise(name):
    g = golden(f"ras_{name}.npz")
    cfg, prob = _cfg_problem(name)
    with threadpool_limits(1, "blas"):
        x, rep = O.newton_ras_solve(prob, np.zeros(2 * cfg.n * cfg.n), cfg.eps0, cfg.gamma,
                                    cfg.eps_min)
    assert rep["converged"] == bool(g["converged"])
    assert rep["outer_iters"] == int(g["outer_iters"])
    assert rep["gmres_iters"] == list(g["gmres_iters"])
    assert rep["alphas"] == list(g["alphas"])
    np.testing.assert_array_equal(rep["residual_norms"], g["residual_norms"])
    n2 = cfg.n * cfg.n
    np.testing.assert_array_equal(x[:n2], g["y"])
    np.testing.assert_array_equal(x[n2:], g["p"])
