"""Parity of the linear-RAS Newton-Krylov path (newton-ras-eps) on the GPU.

Fixtures: ``tests/golden/ras_*.npz`` from the unmodified reference
(``make_golden.py ras_units / ras_cfg1 / ras_cfg2 / ras_cfg3``).

Tolerances: the global residual and Jacobian action follow the reference's
CSR entry order, so they are bitwise for the polynomial phi's and within a
few ulps of the row scale where exp/pow enter (CUDA vs glibc libm).  The RAS
preconditioner solves with a no-pivot block-Thomas elimination instead of SuperLU: relative
1e-10.  Solves: y/p/u within 1e-8 relative L2, outer iterations equal,
GMRES iterations within +-1 per outer step.
"""

import numpy as np
import pytest

import raspen_oracle as O
from conftest import golden
from parity_checks import check_fields
from paper_2411_00546_b200 import (ContinuationSchedule, Grid, KrylovConfig, LocalSolveError,
                                   NewtonConfig, NonfiniteFieldError, ProblemSpec,
                                   build_local_systems, decompose, global_jacobian,
                                   global_residual, make_phi, newton_ras_solve,
                                   ras_precondition, ras_preconditioner)
from paper_2411_00546_b200.linear_ras import GlobalJacobian, RasPreconditioner
from paper_2411_00546_b200.problems import CONFIGS, build_spec, mild_spec
from paper_2411_00546_b200.system import Nonlinearity, recover_control

pytestmark = pytest.mark.gpu

UNIT_CASES = [
    ("kappa16", 16, 2, 2, 2, Nonlinearity(0.1), 1e-2, 1.0),
    ("cubic20", 20, 2, 3, 2, make_phi("cubic"), 1e-3, 1e-2),
    ("expm1_18", 18, 3, 2, 3, make_phi("expm1"), 1e-4, 5e-3),
]
IDS = [c[0] for c in UNIT_CASES]


def unit_spec(n, phi, nu, mu):
    base = mild_spec(n)
    return ProblemSpec(grid=Grid(n), a=None, phi=phi, nu=nu, mu=mu, f=base.f,
                       y_d=10.0 * base.y_d)


def rel_l2(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def ras_cfg(tol=1e-10, sigma=1.1, gmres_tol=1e-8):
    return NewtonConfig(tol=tol, max_outer=200, sigma=sigma,
                        linear_solver=KrylovConfig(rel_tol=gmres_tol, max_iters=2000))


@pytest.fixture(scope="module", autouse=True)
def _native(native_gpu):
    return native_gpu


@pytest.mark.parametrize("case", UNIT_CASES, ids=IDS)
def test_global_residual_and_jacobian_match_reference(case):
    tag, n, s1, s2, m, phi, nu, mu = case
    g = golden("ras_units.npz")
    spec = unit_spec(n, phi, nu, mu)
    eng = build_local_systems(decompose(spec.grid, s1, s2, m), spec)
    x, d, eps = g[f"{tag}_x"], g[f"{tag}_d"], 1e-2
    r = global_residual(eng, x, eps)
    jv = global_jacobian(eng, x, eps)(d)
    for got, ref in ((r, g[f"{tag}_resid"]), (jv, g[f"{tag}_jvp"])):
        if tag.startswith("cubic"):
            np.testing.assert_array_equal(got, ref)
        else:
            np.testing.assert_allclose(got, ref, rtol=0, atol=16e-16 * np.abs(ref).max())


@pytest.mark.parametrize("case", UNIT_CASES, ids=IDS)
def test_ras_preconditioner_matches_reference(case):
    tag, n, s1, s2, m, phi, nu, mu = case
    g = golden("ras_units.npz")
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    out = ras_precondition(g[f"{tag}_d"], g[f"{tag}_x"], dec, spec, 1e-2)
    assert rel_l2(out, g[f"{tag}_prec"]) <= 1e-10
    # device-vector form: same values
    eng = build_local_systems(dec, spec)
    M = ras_preconditioner(eng.from_host(g[f"{tag}_x"]), dec, spec, 1e-2, systems=eng)
    np.testing.assert_array_equal(M(eng.from_host(g[f"{tag}_d"])).to_host(), out)


@pytest.mark.parametrize("case", UNIT_CASES, ids=IDS)
def test_unit_solves_match_reference(case):
    tag, n, s1, s2, m, phi, nu, mu = case
    g = golden("ras_units.npz")
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    x, rep = newton_ras_solve(np.zeros(2 * n * n), dec, spec,
                              ContinuationSchedule(1.0, 0.2, 1e-3), ras_cfg())
    assert rep.converged == bool(g[f"{tag}_solve_converged"])
    assert rep.outer_iters == int(g[f"{tag}_solve_outer"])
    assert rep.alphas == list(g[f"{tag}_solve_alphas"])
    ref_gm = list(g[f"{tag}_solve_gmres"])
    assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_iters, ref_gm))
    assert rel_l2(x, g[f"{tag}_solve_x"]) <= 1e-8


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_baseline_config_ras_solve_matches_reference(name):
    g = golden(f"ras_{name}.npz")
    cfg = CONFIGS[name]
    spec = build_spec(cfg)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    x, rep = newton_ras_solve(np.zeros(2 * cfg.n * cfg.n), dec, spec,
                              ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min), ras_cfg())
    assert rep.converged and bool(g["converged"])
    assert rep.outer_iters == int(g["outer_iters"])
    assert rep.alphas == list(g["alphas"])
    assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_iters, list(g["gmres_iters"])))
    n2 = cfg.n * cfg.n
    y, p = x[:n2], x[n2:]
    u = recover_control(p, spec, cfg.eps_min)
    check_fields(g, {"y": y, "p": p, "u": u}, cfg.mu, cfg.eps_min)


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_large_config_ras_solve_matches_reference(name):
    """Configs 3 (expm1, 8x8) and 4 (headline grid, 16x16): the reference's
    newton-ras-eps record (ras_cfg3: 8 min, ras_cfg4: CPU hours) vs the device."""
    g = golden(f"ras_{name}.npz")
    cfg = CONFIGS[name]
    spec = build_spec(cfg, with_matrix=False)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    x, rep = newton_ras_solve(np.zeros(cfg.unknowns), dec, spec,
                              ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min), ras_cfg())
    assert rep.converged == bool(g["converged"])
    assert rep.outer_iters == int(g["outer_iters"])
    assert rep.alphas == list(g["alphas"])
    assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_iters, list(g["gmres_iters"])))
    n2 = cfg.n * cfg.n
    u = recover_control(x[n2:], spec, cfg.eps_min)
    check_fields(g, {"y": x[:n2], "p": x[n2:], "u": u}, cfg.mu, cfg.eps_min)


def test_fused_preconditioned_gmres_matches_python_gmres():
    """The native left-preconditioned GMRES and the generic device GMRES
    (krylov.gmres with the same operator and preconditioner) agree."""
    from paper_2411_00546_b200.krylov import gmres
    cfg = CONFIGS["cfg1"]
    spec = build_spec(cfg)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    eng = build_local_systems(dec, spec)
    rng = np.random.default_rng(3)
    x = eng.from_host(0.1 * rng.standard_normal(2 * cfg.n * cfg.n))
    b = eng.from_host(rng.standard_normal(2 * cfg.n * cfg.n))
    J = GlobalJacobian(eng, x, 1e-3)
    M = RasPreconditioner(eng, x, 1e-3)
    kc = KrylovConfig(rel_tol=1e-10, max_iters=500)
    fused = J.fused_gmres(b, kc, M)
    plain = gmres(J, b, kc, precond=M)
    assert fused.iters == plain.iters and fused.converged and plain.converged
    assert rel_l2(fused.x.to_host(), plain.x.to_host()) <= 1e-12
    # and it solves J x = b: ||M(J x - b)|| small relative to ||M b||
    mb = M(b).to_host()
    res = M(J(fused.x)).to_host() - mb
    assert np.linalg.norm(res) <= 1e-9 * np.linalg.norm(mb)


def test_nonfinite_jacobian_raises_like_reference():
    n = 12
    spec = unit_spec(n, make_phi("expm1"), 1e-4, 5e-3)
    eng = build_local_systems(decompose(spec.grid, 2, 2, 2), spec)
    x = np.zeros(2 * n * n)
    x[37] = 800.0
    x[5] = 900.0
    with pytest.raises(NonfiniteFieldError) as exc:
        global_jacobian(eng, x, 1e-2)
    assert exc.value.index == 5
    with pytest.raises(NonfiniteFieldError):
        ras_preconditioner(x, decompose(spec.grid, 2, 2, 2), spec, 1e-2, systems=eng)
