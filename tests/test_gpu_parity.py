"""Parity of the CUDA path (through the C ABI) with the oracle and the golden fixtures.

Tolerances: the local residual is evaluated in the reference's rounding
order, so it is compared bitwise for the polynomial phi's and to 4 ulps
(relative 1e-15 of the row scale) where exp/pow are involved (CUDA vs glibc
libm).  Directions / JVPs come from a no-pivot block-Thomas elimination instead of SuperLU:
relative 1e-10.  Solves: BASELINE parity bar, y/p/u within 1e-8 relative L2,
iteration counts within +-1.
"""

import numpy as np
import pytest

import raspen_oracle as O
from conftest import golden
from parity_checks import check_fields
from paper_2411_00546_b200 import (ContinuationSchedule, Grid, KrylovConfig, LocalSolveError,
                                   NewtonConfig, ProblemSpec, build_local_systems, decompose,
                                   make_phi, raspen_jacobian_apply, raspen_residual, raspen_solve)
from paper_2411_00546_b200.problems import CONFIGS, build_spec, mild_spec
from paper_2411_00546_b200.system import Nonlinearity

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


@pytest.fixture(scope="module", autouse=True)
def _native(native_gpu):
    return native_gpu


@pytest.mark.parametrize("case", UNIT_CASES, ids=IDS)
def test_local_residual_matches_oracle(case):
    tag, n, s1, s2, m, phi, nu, mu = case
    g = golden("units.npz")
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    eng = build_local_systems(dec, spec)
    x = g[f"{tag}_x"]
    v = np.concatenate([x[s.pair_idx] + 0.01 for s in dec.subdomains])
    xd, vd, rd = eng.from_host(x), eng.from_host(v), eng.vector(v.shape[0])
    eng.check(eng.lib.ocp_local_residual(eng.ctx, xd.ptr, vd.ptr, 1e-2, rd.ptr), "res")
    r = rd.to_host()
    ref = g[f"{tag}_local_res"]
    if tag.startswith("cubic"):
        np.testing.assert_array_equal(r, ref)
    else:
        scale = np.abs(ref).max()
        np.testing.assert_allclose(r, ref, rtol=0, atol=4e-16 * scale * 4)


@pytest.mark.parametrize("n,s1,s2,m", [(127, 2, 3, 4), (150, 3, 2, 6), (63, 1, 1, 0)])
def test_local_residual_multi_chunk_bitwise(n, s1, s2, m):
    """Subdomains of several 1024-point residual CTAs (halo rows crossing CTA
    boundaries, both orientations, a 1x1 decomposition with no exterior):
    bitwise equal to the oracle's frozen-exterior local residual
    (schwarz.py:174-186) for the cubic phi."""
    phi, nu, mu, eps = make_phi("cubic"), 1e-3, 1e-2, 1e-2
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    eng = build_local_systems(dec, spec)
    prob = O.Problem(n, s1, s2, m, phi, nu, mu, spec.f, spec.y_d)
    rng = np.random.default_rng(7 + n)
    x = 0.3 * rng.standard_normal(2 * n * n)
    v = np.concatenate([x[s.pair_idx] + 0.01 for s in dec.subdomains])
    assert max(s.size for s in dec.subdomains) > 1024
    xd, vd, rd = eng.from_host(x), eng.from_host(v), eng.vector(v.shape[0])
    eng.check(eng.lib.ocp_local_residual(eng.ctx, xd.ptr, vd.ptr, eps, rd.ptr), "res")
    offs = np.cumsum([0] + [2 * s.size for s in dec.subdomains])
    ref = np.concatenate([prob.local_fns(i, x)[0](v[offs[i]:offs[i + 1]], eps)
                          for i in range(len(dec.subdomains))])
    np.testing.assert_array_equal(rd.to_host(), ref)


@pytest.mark.parametrize("n,s1,s2,m", [(127, 2, 3, 4), (63, 1, 1, 0), (40, 3, 2, 5)])
def test_trial_residual_norms_bitwise(n, s1, s2, m):
    """The line-search trial ||F_i(v_i + alpha_i d_i)||^2 (newton.py:96-112) through the
    staged-direction instance of the residual kernel: v + alpha * d with the product
    rounded first, the frozen-exterior local residual of the oracle (schwarz.py:174-186)
    bitwise for the cubic phi, and the squared norm within the summation-order bound
    (per-thread / per-CTA partial sums instead of numpy's pairwise sum)."""
    import ctypes
    phi, nu, mu, eps = make_phi("cubic"), 1e-3, 1e-2, 1e-3
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    eng = build_local_systems(dec, spec)
    prob = O.Problem(n, s1, s2, m, phi, nu, mu, spec.f, spec.y_d)
    rng = np.random.default_rng(11 + n)
    x = 0.3 * rng.standard_normal(2 * n * n)
    v = np.concatenate([x[s.pair_idx] + 0.01 for s in dec.subdomains])
    d = 0.1 * rng.standard_normal(v.shape[0])
    I = len(dec.subdomains)
    alpha = 0.5 ** rng.integers(0, 4, I).astype(float)
    offs = np.cumsum([0] + [2 * s.size for s in dec.subdomains])
    xd, vd, dd = eng.from_host(x), eng.from_host(v), eng.from_host(d)
    out = (ctypes.c_double * I)()
    al = (ctypes.c_double * I)(*alpha)
    eng.check(eng.lib.ocp_local_residual_trial(eng.ctx, xd.ptr, vd.ptr, dd.ptr, al, eps, out), "trial")
    # the same values staged with alpha = 0 give bitwise the same squared norms
    out0 = (ctypes.c_double * I)()
    zero = (ctypes.c_double * I)(*([0.0] * I))
    vt_dev = eng.from_host(np.concatenate([v[offs[i]:offs[i + 1]] + alpha[i] * d[offs[i]:offs[i + 1]]
                                           for i in range(I)]))
    eng.check(eng.lib.ocp_local_residual_trial(eng.ctx, xd.ptr, vt_dev.ptr, dd.ptr, zero, eps, out0), "trial0")
    assert list(out) == list(out0)
    # the staged values feed the same stencil: the residual AT v + alpha d is bitwise the oracle's
    vt = np.concatenate([v[offs[i]:offs[i + 1]] + alpha[i] * d[offs[i]:offs[i + 1]] for i in range(I)])
    rd = eng.vector(v.shape[0])
    eng.check(eng.lib.ocp_local_residual(eng.ctx, xd.ptr, eng.from_host(vt).ptr, eps, rd.ptr), "res")
    r = rd.to_host()
    for i in range(I):
        ref = prob.local_fns(i, x)[0](vt[offs[i]:offs[i + 1]], eps)
        np.testing.assert_array_equal(r[offs[i]:offs[i + 1]], ref)
        want = float(np.dot(ref, ref))
        assert abs(out[i] - want) <= 1e-13 * want, (i, out[i], want)


@pytest.mark.parametrize("case", UNIT_CASES, ids=IDS)
def test_local_direction_matches_superlu(case):
    import scipy.sparse.linalg as spla
    tag, n, s1, s2, m, phi, nu, mu = case
    g = golden("units.npz")
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    eng = build_local_systems(dec, spec)
    prob = O.Problem(n, s1, s2, m, phi, nu, mu, spec.f, spec.y_d)
    x = g[f"{tag}_x"]
    v = np.concatenate([x[s.pair_idx] + 0.01 for s in dec.subdomains])
    xd, vd, dd = eng.from_host(x), eng.from_host(v), eng.vector(v.shape[0])
    eng.check(eng.lib.ocp_local_direction(eng.ctx, xd.ptr, vd.ptr, 1e-2, dd.ptr), "dir")
    d = dd.to_host()
    off = 0
    for i, s in enumerate(dec.subdomains):
        F, J = prob.local_fns(i, x)
        vi = x[s.pair_idx] + 0.01
        ref = spla.splu(J(vi, 1e-2).tocsc()).solve(-F(vi, 1e-2))
        got = d[off:off + 2 * s.size]
        assert rel_l2(got, ref) <= 1e-10, (i, rel_l2(got, ref))
        off += 2 * s.size


@pytest.mark.parametrize("case", UNIT_CASES, ids=IDS)
def test_raspen_residual_and_jvp_match_golden(case):
    tag, n, s1, s2, m, phi, nu, mu = case
    g = golden("units.npz")
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    x = g[f"{tag}_x"]
    f_val, corr = raspen_residual(x, dec, spec, 1e-2, inner_cfg=NewtonConfig(tol=1e-10))
    assert corr.inner_iters == list(g[f"{tag}_inner"])
    assert rel_l2(f_val, g[f"{tag}_fval"]) <= 1e-10
    out = raspen_jacobian_apply(x, g[f"{tag}_d"], dec, spec, 1e-2, corr)
    assert rel_l2(out, g[f"{tag}_jvp"]) <= 1e-10


@pytest.mark.parametrize("case", UNIT_CASES, ids=IDS)
def test_raspen_solve_matches_golden(case):
    tag, n, s1, s2, m, phi, nu, mu = case
    g = golden("units.npz")
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    x, rep = raspen_solve(np.zeros(2 * n * n), dec, spec, ContinuationSchedule(1.0, 0.2, 1e-3),
                          cfg=NewtonConfig(tol=1e-10),
                          krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000))
    assert rep.converged == bool(g[f"{tag}_solve_converged"])
    assert rel_l2(x, g[f"{tag}_solve_x"]) <= 1e-8
    assert abs(rep.outer_iters - int(g[f"{tag}_solve_outer"])) <= 1
    ref_inner = list(g[f"{tag}_solve_inner"])
    for a, b in zip(rep.inner_iters, ref_inner):
        assert abs(a - b) <= 1
    for a, b in zip(rep.gmres_iters, list(g[f"{tag}_solve_gmres"])):
        assert abs(a - b) <= 1


def _check_solve_record(name, g, x, rep, cfg):
    n2 = cfg.n * cfg.n
    y, p = x[:n2], x[n2:]
    from paper_2411_00546_b200.system import recover_control
    spec = build_spec(cfg, with_matrix=False)
    u = recover_control(p, spec, cfg.eps_min)
    assert rep.converged == bool(g["converged"]), rep.failure
    assert abs(rep.outer_iters - int(g["outer_iters"])) <= 1
    for a, b in zip(rep.inner_iters, list(g["inner_iters"])):
        assert abs(a - b) <= 1, (rep.inner_iters, list(g["inner_iters"]))
    for a, b in zip(rep.gmres_iters, list(g["gmres_iters"])):
        assert abs(a - b) <= 1, (rep.gmres_iters, list(g["gmres_iters"]))
    check_fields(g, {"y": y, "p": p, "u": u}, cfg.mu, cfg.eps_min)


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_baseline_config_solve_matches_reference(name):
    g = golden(f"{name}_tol1e-08.npz")
    cfg = CONFIGS[name]
    spec = build_spec(cfg, with_matrix=False)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    x, rep = raspen_solve(np.zeros(cfg.unknowns), dec, spec,
                          ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min),
                          cfg=NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1),
                          krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000), inner_tol=1e-8)
    _check_solve_record(name, g, x, rep, cfg)
    ref_ps = g["per_sub"]
    got_ps = np.array(rep.per_subdomain_inner)
    assert got_ps.shape == ref_ps.shape
    assert np.abs(got_ps - ref_ps).max() <= 1


def _solve_cfg(name, inner_tol):
    cfg = CONFIGS[name]
    spec = build_spec(cfg, with_matrix=False)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    x, rep = raspen_solve(np.zeros(cfg.unknowns), dec, spec,
                          ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min),
                          cfg=NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1),
                          krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000),
                          inner_tol=inner_tol)
    return cfg, x, rep


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_deviation_solve_matches_reference(name):
    """Configs 3/4 at the documented deviation inner_tol = 1e-7 (both arms)."""
    g = golden(f"{name}_tol1e-07.npz")
    cfg, x, rep = _solve_cfg(name, 1e-7)
    _check_solve_record(name, g, x, rep, cfg)


def test_cfg3_reference_settings_fail_like_the_reference():
    """At inner_tol = 1e-8 the reference fails config 3 (FP64 residual floor,
    SURVEY 0.13); the GPU path must fail the same way: LocalSolveError in the
    same evaluation, a stalling subdomain, x0 returned."""
    g = golden("cfg3_tol1e-08.npz")
    cfg, x, rep = _solve_cfg("cfg3", 1e-8)
    assert not rep.converged and not bool(g["converged"])
    assert "subdomain" in rep.failure and "no convergence within 200" in rep.failure
    failed = int(rep.failure.split()[1].rstrip(":"))
    ref_failed = int(str(g["failure"]).split()[1].rstrip(":"))
    assert ref_failed == 38
    assert failed == ref_failed, (rep.failure, str(g["failure"]))
    assert rep.failure == str(g["failure"])
    assert rep.outer_iters == int(g["outer_iters"])
    assert len(rep.inner_iters) == len(g["inner_iters"])
    for a, b in zip(rep.inner_iters, list(g["inner_iters"])):
        assert abs(a - b) <= 1
    np.testing.assert_array_equal(x, np.zeros(cfg.unknowns))


def test_cfg4_reference_settings_fail_like_the_reference():
    """The headline config at the reference's own inner_tol = 1e-8: the
    reference fails in the third RAS evaluation with subdomain 39 stalling at
    the FP64 residual floor (tests/golden/cfg4_tol1e-08.npz, 56 min on the CPU);
    the GPU path reproduces the same record."""
    g = golden("cfg4_tol1e-08.npz")
    cfg, x, rep = _solve_cfg("cfg4", 1e-8)
    assert not rep.converged and not bool(g["converged"])
    assert rep.failure == str(g["failure"])
    assert rep.outer_iters == int(g["outer_iters"])
    assert rep.inner_iters == list(g["inner_iters"])
    np.testing.assert_array_equal(x, np.zeros(cfg.unknowns))


@pytest.mark.parametrize("name", ["cfg5u", "cfg5"])
def test_cfg5_sweep_and_jvp_match_reference(name):
    from paper_2411_00546_b200.schwarz import _jvp, _sweep
    g = golden(f"{name}_sweep.npz")
    cfg = CONFIGS[name]
    spec = build_spec(cfg, with_matrix=False)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    eng = build_local_systems(dec, spec)
    x = eng.from_host(np.zeros(cfg.unknowns))
    fac = eng.factor_store()
    fval, inner = _sweep(eng, x, fac, ContinuationSchedule.fixed(cfg.eps_min),
                         NewtonConfig(tol=1e-8, max_outer=200))
    assert inner == list(g["inner_iters"])
    d = eng.from_host(np.random.default_rng(1).standard_normal(cfg.unknowns))
    out = _jvp(eng, fac, d).to_host()
    fv = fval.to_host()
    for key, vec in (("fval", fv), ("jvp", out)):
        stride = int(g[f"{key}_stride"])
        assert rel_l2(vec[::stride], g[f"{key}_samples"]) <= 1e-10, key
        assert abs(np.linalg.norm(vec) - float(g[f"{key}_norm"])) <= 1e-10 * float(g[f"{key}_norm"])


@pytest.mark.parametrize("n,parts,m", [(400, 20, 2), (360, 18, 4), (320, 20, 2), (395, 18, 3), (60, 20, 1)])
def test_many_small_subdomains_sweep_and_jvp_match_oracle(n, parts, m):
    """Decompositions of >= 2 subdomains per SM run the narrow-line factor instance
    (ocp_block_narrow.cu): lines padded to 16 with a half-width last panel (local sides
    24 / 28 -> 48 / 56 unknowns at NPB = 48 / 64, uneven tilings with larger last tiles
    that go to the 12-warp kernel on the second stream), lines that are a multiple of 32
    (54 unknowns at NPB = 64), and an 82-unknown corner (n = 395: 17 tiles of 21 and one of 38)
    beyond the instance (12-warp kernel, second stream).  One RAS sweep at fixed
    eps and one JVP against the oracle's SuperLU path (schwarz.py:285-345)."""
    from paper_2411_00546_b200.schwarz import _jvp, _sweep
    phi, nu, mu, eps = make_phi("cubic"), 1e-3, 1e-2, 1e-3
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, parts, parts, m)
    assert len(dec.subdomains) >= 296
    eng = build_local_systems(dec, spec)
    prob = O.Problem(n, parts, parts, m, phi, nu, mu, spec.f, spec.y_d)
    x0 = np.zeros(2 * n * n)
    x = eng.from_host(x0)
    fac = eng.factor_store()
    fval, inner = _sweep(eng, x, fac, ContinuationSchedule.fixed(eps), NewtonConfig(tol=1e-8, max_outer=200))
    f_ref, corr = O.raspen_residual(prob, x0, eps, tol=1e-8, threads=8)
    assert inner == corr.inner
    assert rel_l2(fval.to_host(), f_ref) <= 1e-10
    d = np.random.default_rng(5).standard_normal(2 * n * n)
    out = _jvp(eng, fac, eng.from_host(d)).to_host()
    assert rel_l2(out, O.raspen_jvp(prob, x0, d, eps, corr)) <= 1e-10


def test_jvp_properties_linear_zero_and_single_domain_identity():
    """Reference property tests (`test_schwarz.py:285-308`) on the device path."""
    tag, n, s1, s2, m, phi, nu, mu = UNIT_CASES[0]
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    rng = np.random.default_rng(33)
    x = 0.2 * rng.standard_normal(2 * n * n)
    _, corr = raspen_residual(x, dec, spec, 1e-2, inner_cfg=NewtonConfig(tol=1e-12))
    apply = lambda d: raspen_jacobian_apply(x, d, dec, spec, 1e-2, corr)  # noqa: E731
    np.testing.assert_array_equal(apply(np.zeros_like(x)), np.zeros_like(x))
    d1, d2 = rng.standard_normal((2, x.shape[0]))
    np.testing.assert_allclose(apply(3.0 * d1 + d2), 3.0 * apply(d1) + apply(d2),
                               rtol=1e-11, atol=1e-11)
    dec1 = decompose(spec.grid, 1, 1, 0)
    _, corr1 = raspen_residual(x, dec1, spec, 1e-2, inner_cfg=NewtonConfig(tol=1e-13))
    d = rng.standard_normal(x.shape)
    out = raspen_jacobian_apply(x, d, dec1, spec, 1e-2, corr1)
    np.testing.assert_allclose(out, -d, rtol=1e-9, atol=1e-9)


def test_jvp_matches_finite_differences():
    """`test_schwarz.py:310-323`: directional FD of the fixed-point residual."""
    tag, n, s1, s2, m, phi, nu, mu = UNIT_CASES[0]
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    rng = np.random.default_rng(37)
    x = 0.1 * rng.standard_normal(2 * n * n)
    tight = NewtonConfig(tol=1e-12)
    f0, corr = raspen_residual(x, dec, spec, 1e-2, inner_cfg=tight)
    tau = 1e-5
    for _ in range(3):
        d = rng.standard_normal(x.shape)
        d /= np.linalg.norm(d)
        f1, _ = raspen_residual(x + tau * d, dec, spec, 1e-2, inner_cfg=tight)
        fd = (f1 - f0) / tau
        jd = raspen_jacobian_apply(x, d, dec, spec, 1e-2, corr)
        assert np.linalg.norm(fd - jd) <= 1e-4 * max(1.0, np.linalg.norm(jd))


def test_stale_corrections_rejected():
    tag, n, s1, s2, m, phi, nu, mu = UNIT_CASES[0]
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    x = np.zeros(2 * n * n)
    _, corr = raspen_residual(x, dec, spec, 1e-2)
    with pytest.raises(RuntimeError, match="stale"):
        raspen_jacobian_apply(x + 1.0, np.ones_like(x), dec, spec, 1e-2, corr)
    with pytest.raises(RuntimeError, match="stale"):
        raspen_jacobian_apply(x, np.ones_like(x), dec, spec, 1e-3, corr)


def test_local_failure_becomes_failed_report_and_solve_is_deterministic():
    tag, n, s1, s2, m, phi, nu, mu = UNIT_CASES[1]
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    sched = ContinuationSchedule(1.0, 0.2, 1e-3)
    x0 = np.zeros(2 * n * n)
    x, rep = raspen_solve(x0, dec, spec, sched, inner_max_outer=0)
    assert not rep.converged and "subdomain" in rep.failure
    np.testing.assert_array_equal(x, x0)
    xa, ra = raspen_solve(x0, dec, spec, sched, threads=1)
    xb, rb = raspen_solve(x0, dec, spec, sched, threads=2)
    assert ra.converged and rb.converged
    np.testing.assert_array_equal(xa, xb)
    assert ra.residual_norms == rb.residual_norms
    assert len(ra.inner_iters) == ra.outer_iters + 1 and set(ra.alphas) == {1.0}


def test_fused_native_gmres_matches_python_gmres():
    """The native GMRES (ocp_raspen_gmres) and the Python device GMRES run the
    same algorithm on the same operator: same iteration count, history to
    rounding, solution to 1e-12."""
    from paper_2411_00546_b200 import gmres
    from paper_2411_00546_b200.schwarz import _RaspenOperator, _sweep
    tag, n, s1, s2, m, phi, nu, mu = UNIT_CASES[1]
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    eng = build_local_systems(dec, spec)
    rng = np.random.default_rng(7)
    xd = eng.from_host(0.2 * rng.standard_normal(2 * n * n))
    fac = eng.factor_store()
    fval, _ = _sweep(eng, xd, fac, ContinuationSchedule.fixed(1e-2), NewtonConfig(tol=1e-10))
    state = {"corr": "c"}
    op = _RaspenOperator(eng, fac, state, "c")
    b = fval.scaled(-1.0)
    cfg = KrylovConfig(rel_tol=1e-10, max_iters=200)
    r1 = gmres(op, b, cfg)
    r2 = op.fused_gmres(b, cfg)
    assert r1.converged and r2.converged and r1.iters == r2.iters
    np.testing.assert_allclose(r2.history, r1.history, rtol=1e-10)
    assert rel_l2(r2.x.to_host(), r1.x.to_host()) <= 1e-12


@pytest.mark.gpu
def test_fresh_contexts_reuse_memory_and_agree_bitwise():
    """Solves on successive fresh contexts (device buffers retired to the
    process cache, the GMRES basis from the stream-ordered pool) give
    bitwise-identical iterates and reports."""
    import gc
    cfg = CONFIGS["cfg2"]
    spec = build_spec(cfg, with_matrix=False)
    res = []
    for _ in range(3):
        fresh = type(spec)(grid=spec.grid, a=None, phi=spec.phi, nu=spec.nu, mu=spec.mu,
                           f=spec.f.copy(), y_d=spec.y_d.copy())
        dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
        x, rep = raspen_solve(np.zeros(cfg.unknowns), dec, fresh,
                              ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min),
                              cfg=NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1),
                              krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000), inner_tol=1e-8)
        res.append((x, rep.gmres_iters, rep.inner_iters))
        del dec, fresh
        gc.collect()
    for x, g_it, i_it in res[1:]:
        np.testing.assert_array_equal(x, res[0][0])
        assert g_it == res[0][1] and i_it == res[0][2]


VARIANT_CASES = [("kappa16",) + UNIT_CASES[0][1:], ("cubic20",) + UNIT_CASES[1][1:]]


def _variant_problem(tag):
    if tag == "cfg1":
        cfg = CONFIGS["cfg1"]
        spec = build_spec(cfg, with_matrix=False)
        return (spec, decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap),
                ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min))
    case = dict((c[0], c) for c in VARIANT_CASES)[tag]
    _, n, s1, s2, m, phi, nu, mu = case
    spec = unit_spec(n, phi, nu, mu)
    return spec, decompose(spec.grid, s1, s2, m), ContinuationSchedule(1.0, 0.2, 1e-3)


@pytest.mark.parametrize("tag", ["kappa16", "cubic20", "cfg1"])
@pytest.mark.parametrize("var", ["nocont", "backtrack"])
def test_solve_variants_match_reference(tag, var):
    """raspen_solve(continuation=False) (`pkg/tests/test_schwarz.py:350-358`)
    and raspen_solve(backtracking=True) (sigma = 1.1 outer line search,
    `schwarz.py:397-401`) against the unmodified reference's records
    (tests/golden/variants.npz): same iteration counts, step lengths and
    per-subdomain inner counts, iterate within 1e-8."""
    g = golden("variants.npz")
    k = f"{tag}_{var}"
    spec, dec, sched = _variant_problem(tag)
    kw = dict(continuation=False) if var == "nocont" else dict(backtracking=True)
    x, rep = raspen_solve(np.zeros(2 * spec.grid.size), dec, spec, sched,
                          cfg=NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1),
                          krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000), **kw)
    assert rep.converged == bool(g[f"{k}_converged"])
    assert rep.outer_iters == int(g[f"{k}_outer"])
    assert rep.inner_iters == list(g[f"{k}_inner"])
    assert rep.alphas == list(g[f"{k}_alphas"])
    assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_iters, list(g[f"{k}_gmres"])))
    ref_ps = g[f"{k}_per_sub"]
    assert np.array(rep.per_subdomain_inner).shape == ref_ps.shape
    assert np.abs(np.array(rep.per_subdomain_inner) - ref_ps).max() <= 1
    assert rel_l2(x, g[f"{k}_x"]) <= 1e-8
    np.testing.assert_allclose(rep.residual_norms, g[f"{k}_norms"], rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("tag", ["kappa16", "cubic20"])
def test_residual_with_inner_schedule_floor_below_eps(tag):
    """raspen_residual with an inner schedule whose floor (1e-3) differs from
    eps (1e-2): the reference solves the local problems along the schedule and
    then refactors at eps (`schwarz.py:296-315`); f_val, inner counts and the
    JVP from the stored factors match its record."""
    g = golden("variants.npz")
    spec, dec, _ = _variant_problem(tag)
    x = g[f"{tag}_floor_x"]
    f_val, corr = raspen_residual(x, dec, spec, 1e-2, inner_cfg=NewtonConfig(tol=1e-10),
                                  inner_sched=ContinuationSchedule(1.0, 0.2, 1e-3))
    assert corr.inner_iters == list(g[f"{tag}_floor_inner"])
    assert rel_l2(f_val, g[f"{tag}_floor_fval"]) <= 1e-10
    out = raspen_jacobian_apply(x, g[f"{tag}_floor_d"], dec, spec, 1e-2, corr)
    assert rel_l2(out, g[f"{tag}_floor_jvp"]) <= 1e-10


@pytest.mark.parametrize("tag", ["kappa16", "cubic20"])
def test_local_correction_single_subdomain(tag):
    """local_correction(i) (`schwarz.py:211-218`) solves subdomain i alone."""
    from paper_2411_00546_b200 import local_correction
    g = golden("variants.npz")
    spec, dec, _ = _variant_problem(tag)
    x = g[f"{tag}_floor_x"]
    for i in (0, len(dec) - 1):
        v = local_correction(i, x, dec, spec, 1e-2, inner_cfg=NewtonConfig(tol=1e-10))
        assert rel_l2(v, g[f"{tag}_lc{i}"]) <= 1e-10


def test_correction_set_jac_locs_are_the_local_jacobians():
    """CorrectionSet.jac_locs[i] is the local Jacobian at the corrected values
    (`schwarz.py:166-171,321`), equal to the oracle's assembly."""
    import scipy.sparse.linalg  # noqa: F401
    tag, n, s1, s2, m, phi, nu, mu = UNIT_CASES[1]
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    prob = O.Problem(n, s1, s2, m, phi, nu, mu, spec.f, spec.y_d)
    x = 0.2 * np.random.default_rng(5).standard_normal(2 * n * n)
    _, corr = raspen_residual(x, dec, spec, 1e-2, inner_cfg=NewtonConfig(tol=1e-10))
    assert len(corr.jac_locs) == len(dec)
    for i in range(len(dec)):
        J = corr.jac_locs[i]
        Jo = prob.local_fns(i, x)[1](corr.values[i], 1e-2)
        d = np.random.default_rng(i).standard_normal(J.shape[0])
        np.testing.assert_allclose(J @ d, Jo @ d, rtol=1e-13, atol=1e-9)


def test_small_context_does_not_shrink_kernel_limits_of_a_larger_one():
    """Kernel shared-memory limits are process-wide: a context of small
    subdomains created after a larger one must not break the larger one's
    launches (regression: cudaErrorInvalidValue from k_residual)."""
    from paper_2411_00546_b200.schwarz import _sweep
    cfg = CONFIGS["cfg2"]
    spec = build_spec(cfg, with_matrix=False)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    big = build_local_systems(dec, spec)
    tag, n, s1, s2, m, phi, nu, mu = UNIT_CASES[0]
    small_spec = unit_spec(n, phi, nu, mu)
    build_local_systems(decompose(small_spec.grid, s1, s2, m), small_spec)
    x = big.from_host(np.zeros(cfg.unknowns))
    _, inner = _sweep(big, x, big.factor_store(), ContinuationSchedule.fixed(1e-3),
                      NewtonConfig(tol=1e-8))
    assert max(inner) >= 1


@pytest.mark.parametrize("case", UNIT_CASES[:2], ids=IDS[:2])
def test_native_gmres_matches_oracle_gmres(case):
    """The native GMRES (lagged-dot MGS Arnoldi on the device, Givens on the
    host) against the oracle's restatement of `krylov.py:44-151` on the
    RASPEN Jacobian action at the same iterate: same iteration count, the
    residual history and the direction to 1e-9 (the MGS coefficients are
    summed in a different order; the operators agree to ~1e-13)."""
    from paper_2411_00546_b200.schwarz import _RaspenOperator, _sweep
    tag, n, s1, s2, m, phi, nu, mu = case
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    eng = build_local_systems(dec, spec)
    prob = O.Problem(n, s1, s2, m, phi, nu, mu, spec.f, spec.y_d)
    x = 0.2 * np.random.default_rng(41).standard_normal(2 * n * n)
    eps = 1e-2
    fac = eng.factor_store()
    fval, _ = _sweep(eng, eng.from_host(x), fac, ContinuationSchedule.fixed(eps),
                     NewtonConfig(tol=1e-12))
    op = _RaspenOperator(eng, fac, {"corr": "c"}, "c")
    cfg = KrylovConfig(rel_tol=1e-10, max_iters=300)
    got = op.fused_gmres(fval.scaled(-1.0), cfg)
    fo, co = O.raspen_residual(prob, x, eps, tol=1e-12, threads=1)
    do, ko, ro, cvo, ho = O.gmres(lambda v: O.raspen_jvp(prob, x, v, eps, co), -fo, 1e-10, 300)
    assert got.converged and cvo
    assert got.iters == ko, (got.iters, ko)
    h0 = ho[0]
    assert np.max(np.abs(np.array(got.history) - np.array(ho)) / h0) <= 1e-9
    assert rel_l2(got.x.to_host(), do) <= 1e-9


def test_device_gmres_on_the_global_jacobian_matches_oracle():
    """krylov.gmres on device vectors with the global Jacobian J(x) (bitwise
    the reference's `jacobian(x) @ d`, `system.py:155-160`) against the
    oracle's gmres on the same CSR operator (config 1)."""
    from paper_2411_00546_b200 import gmres
    from paper_2411_00546_b200.linear_ras import GlobalJacobian
    cfg = CONFIGS["cfg1"]
    spec = build_spec(cfg)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    eng = build_local_systems(dec, spec)
    rng = np.random.default_rng(5)
    x = 0.1 * rng.standard_normal(cfg.unknowns)
    b = rng.standard_normal(cfg.unknowns)
    J = GlobalJacobian(eng, eng.from_host(x), 1e-3)
    prob = O.Problem(cfg.n, cfg.s1, cfg.s2, cfg.overlap, spec.phi, spec.nu, spec.mu, spec.f, spec.y_d)
    Jo = O.global_jacobian(prob, x, 1e-3)
    kc = KrylovConfig(rel_tol=1e-10, max_iters=400)
    got = gmres(J, eng.from_host(b), kc)
    do, ko, ro, cvo, ho = O.gmres(lambda v: Jo @ v, b, 1e-10, 400)
    assert got.iters == ko and got.converged == cvo
    assert np.max(np.abs(np.array(got.history) - np.array(ho)) / ho[0]) <= 1e-10
    assert rel_l2(got.x.to_host(), do) <= 1e-9


def test_local_correction_ignores_other_subdomains_failures():
    """With an inner iteration budget that only some subdomains meet,
    raspen_residual raises the lowest failing subdomain (the reference's
    thread-pool map), while local_correction(i) of a subdomain within the
    budget returns its values (`schwarz.py:211-218` solves i alone)."""
    from paper_2411_00546_b200 import local_correction
    tag, n, s1, s2, m, phi, nu, mu = UNIT_CASES[1]
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    prob = O.Problem(n, s1, s2, m, phi, nu, mu, spec.f, spec.y_d)
    x = 0.3 * np.random.default_rng(17).standard_normal(2 * n * n)
    sched = ContinuationSchedule(1.0, 0.2, 1e-2)
    counts = [prob.local_solve(i, x, 1.0, 0.2, 1e-2, 1e-10, 200)[1] for i in range(len(dec))]
    budget = min(counts)
    assert max(counts) > budget, counts   # some subdomain needs more than the budget
    ok = counts.index(budget)
    cfg = NewtonConfig(tol=1e-10, max_outer=budget)
    with pytest.raises(LocalSolveError) as exc:
        raspen_residual(x, dec, spec, 1e-2, inner_cfg=cfg, inner_sched=sched)
    assert exc.value.subdomain == next(i for i, c in enumerate(counts) if c > budget)
    v = local_correction(ok, x, dec, spec, 1e-2, inner_cfg=cfg, inner_sched=sched)
    vo, _ = prob.local_solve(ok, x, 1.0, 0.2, 1e-2, 1e-10, budget)
    assert rel_l2(v, vo) <= 1e-10


@pytest.mark.parametrize("n,s1,s2,m", [(4, 2, 2, 0), (5, 2, 1, 1), (7, 3, 3, 1), (9, 1, 3, 2), (6, 1, 1, 0)])
def test_tiny_grids_residual_and_jvp_match_oracle(n, s1, s2, m):
    """Edge cases of the tiling: tiny grids, zero overlap, 1-wide owned tiles,
    single subdomain - RAS residual and JVP against the oracle."""
    phi, nu, mu = make_phi("cubic"), 1e-3, 1e-2
    spec = unit_spec(n, phi, nu, mu)
    dec = decompose(spec.grid, s1, s2, m)
    prob = O.Problem(n, s1, s2, m, phi, nu, mu, spec.f, spec.y_d)
    rng = np.random.default_rng(n * 10 + s1)
    x = 0.2 * rng.standard_normal(2 * n * n)
    f_val, corr = raspen_residual(x, dec, spec, 1e-2, inner_cfg=NewtonConfig(tol=1e-11))
    fo, co = O.raspen_residual(prob, x, 1e-2, tol=1e-11, threads=1)
    assert corr.inner_iters == list(co.inner)
    assert rel_l2(f_val, fo) <= 1e-10
    d = rng.standard_normal(x.shape[0])
    out = raspen_jacobian_apply(x, d, dec, spec, 1e-2, corr)
    assert rel_l2(out, O.raspen_jvp(prob, x, d, 1e-2, co)) <= 1e-10


@pytest.mark.gpu
def test_branch_free_division_and_sqrt_are_bitwise_ieee():
    """div_fast / sqrt_fast / dvd_const_fast of the local residual (ocp_common.cuh) against
    __ddiv_rn / __dsqrt_rn: random, near-tie and residual-shaped operands, 4e9 comparisons
    (tools/rn_check.cu; exit code 1 on any mismatch)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "rn_check")
    if not os.path.exists(exe):
        from paper_2411_00546_b200._build import build_tools
        build_tools()
    out = subprocess.run([exe, "1024"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches div 0, sqrt 0, dvd_const 0, near-tie 0" in out.stdout, out.stdout
