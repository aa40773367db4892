"""Decompositions whose local short side exceeds the fast kernels' 112 points.

The reference factors any local Jacobian with SuperLU (`schwarz.py:305-315`,
`newton.py:125-129`); here lines wider than 224 unknowns run the factor with
its Schur rows in an L2 scratch and the solve on ``k_block_solve_wide``.
Checked against SuperLU / the oracle on random iterates and against fixtures
made by the unmodified reference (tests/golden/wide.npz):

* ``wide2x2``: raspen_solve on 300^2, 2x2 subdomains, overlap 8 (short side 158);
* ``mono150``: monolithic newton-eps with the direct direction on 150^2
  (one block factor of the whole grid: 300-unknown lines).
"""

import ctypes

import numpy as np
import pytest

import raspen_oracle as O
from conftest import golden
from parity_checks import check_fields, rel_l2
from paper_2411_00546_b200 import (ContinuationSchedule, KrylovConfig, NewtonConfig,
                                   build_local_systems, decompose, newton_continuation,
                                   raspen_jacobian_apply, raspen_residual, raspen_solve)
from paper_2411_00546_b200.linear_ras import GlobalJacobian, global_residual
from paper_2411_00546_b200.problems import EXTRA_CONFIGS, build_spec
from paper_2411_00546_b200.system import recover_control

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _native(native_gpu):
    return native_gpu


def _problem(name):
    cfg = EXTRA_CONFIGS[name]
    spec = build_spec(cfg, with_matrix=False)
    return cfg, spec, decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)


def test_wide_decomposition_is_wide():
    cfg, spec, dec = _problem("wide2x2")
    eng = build_local_systems(dec, spec)
    assert min(int(r[10]) for r in eng.rects) > 112   # every short side beyond the fast path


@pytest.mark.parametrize("n,s1,s2,m", [(300, 2, 2, 8), (250, 1, 2, 3)])
def test_wide_local_direction_matches_superlu(n, s1, s2, m):
    import scipy.sparse.linalg as spla
    from paper_2411_00546_b200 import Grid, ProblemSpec, make_phi
    from paper_2411_00546_b200.problems import mild_spec
    base = mild_spec(n)
    spec = ProblemSpec(grid=Grid(n), a=None, phi=make_phi("cubic"), nu=1e-3, mu=1e-2,
                       f=base.f, y_d=10.0 * base.y_d)
    dec = decompose(spec.grid, s1, s2, m)
    eng = build_local_systems(dec, spec)
    prob = O.Problem(n, s1, s2, m, spec.phi, spec.nu, spec.mu, spec.f, spec.y_d)
    x = 0.3 * np.random.default_rng(11).standard_normal(2 * n * n)
    v = np.concatenate([x[s.pair_idx] + 0.01 for s in dec.subdomains])
    xd, vd, dd = eng.from_host(x), eng.from_host(v), eng.vector(v.shape[0])
    eng.check(eng.lib.ocp_local_direction(eng.ctx, xd.ptr, vd.ptr, 1e-2, dd.ptr), "dir")
    d = dd.to_host()
    off = 0
    for i, s in enumerate(dec.subdomains):
        F, J = prob.local_fns(i, x)
        vi = x[s.pair_idx] + 0.01
        ref = spla.splu(J(vi, 1e-2).tocsc()).solve(-F(vi, 1e-2))
        assert rel_l2(d[off:off + 2 * s.size], ref) <= 1e-10, i
        off += 2 * s.size


def test_wide_raspen_residual_and_jvp_match_oracle():
    cfg, spec, dec = _problem("wide2x2")
    prob = O.Problem(cfg.n, cfg.s1, cfg.s2, cfg.overlap, spec.phi, spec.nu, spec.mu, spec.f, spec.y_d)
    rng = np.random.default_rng(21)
    x = 0.2 * rng.standard_normal(cfg.unknowns)
    f_val, corr = raspen_residual(x, dec, spec, 1e-2, inner_cfg=NewtonConfig(tol=1e-10))
    fo, co = O.raspen_residual(prob, x, 1e-2, tol=1e-10, threads=4)
    assert corr.inner_iters == list(co.inner)
    assert rel_l2(f_val, fo) <= 1e-10
    d = rng.standard_normal(cfg.unknowns)
    out = raspen_jacobian_apply(x, d, dec, spec, 1e-2, corr)
    assert rel_l2(out, O.raspen_jvp(prob, x, d, 1e-2, co)) <= 1e-10


def _check(g, tag, cfg, x, rep):
    assert rep.converged == bool(g[f"{tag}_converged"])
    assert abs(rep.outer_iters - int(g[f"{tag}_outer"])) <= 1
    for a, b in zip(rep.gmres_iters, list(g[f"{tag}_gmres"])):
        assert b < 0 or abs(a - b) <= 1
    n2 = cfg.n * cfg.n
    spec = build_spec(cfg, with_matrix=False)
    u = recover_control(x[n2:], spec, cfg.eps_min)

    class View:   # the fixture's per-tag keys under check_fields' names
        files = [k[len(tag) + 1:] for k in g.files if k.startswith(tag + "_")]

        def __getitem__(self, k):
            return g[f"{tag}_{k}"]
    check_fields(View(), {"y": x[:n2], "p": x[n2:], "u": u}, cfg.mu, cfg.eps_min)


def test_wide_raspen_solve_matches_reference():
    g = golden("wide.npz")
    cfg, spec, dec = _problem("wide2x2")
    x, rep = raspen_solve(np.zeros(cfg.unknowns), dec, spec,
                          ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min),
                          cfg=NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1),
                          krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000), inner_tol=1e-8)
    _check(g, "wide2x2", cfg, x, rep)
    for a, b in zip(rep.inner_iters, list(g["wide2x2_inner"])):
        assert abs(a - b) <= 1
    assert np.abs(np.array(rep.per_subdomain_inner) - g["wide2x2_per_sub"]).max() <= 1


def test_monolithic_direct_newton_beyond_112_matches_reference():
    """newton-eps with the direct direction (`harness/experiments.py:86-91`,
    `newton.py:125-129`) on a 150^2 grid: one block factor of the whole
    Jacobian per Newton step (300-unknown lines)."""
    g = golden("wide.npz")
    cfg, spec, dec = _problem("mono150")
    eng = build_local_systems(dec, spec)
    x, rep = newton_continuation(
        eng.from_host(np.zeros(cfg.unknowns)), lambda x, eps: global_residual(eng, x, eps),
        lambda x, eps: GlobalJacobian(eng, x, eps),
        ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min),
        NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1, linear_solver="direct"))
    assert rep.alphas == list(g["mono150_alphas"])
    _check(g, "mono150", cfg, x.to_host(), rep)


def test_multi_cta_paths_match_the_single_cta_paths(monkeypatch):
    """k_block_factor_mc (K CTAs per wide subdomain, default for few
    subdomains) stores exactly the single-CTA factor's -W_a (bitwise, via the
    RAS preconditioner's factorisation at fixed values); k_block_solve_mc
    sums the K partial rows in rank order, so its solves agree to rounding."""
    from paper_2411_00546_b200.linear_ras import RasPreconditioner
    cfg, spec, _ = _problem("wide2x2")
    rng = np.random.default_rng(2)
    x = 0.1 * rng.standard_normal(cfg.unknowns)
    v = rng.standard_normal(cfg.unknowns)
    out = {}
    for mc in ("1", "0"):
        monkeypatch.setenv("OCP_FACTOR_MC", mc)
        dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)   # fresh engine
        eng = build_local_systems(dec, spec)
        M = RasPreconditioner(eng, eng.from_host(x), 1e-3)
        store = np.empty(eng.fac_len)
        eng.check(eng.lib.ocp_d2h(eng.ctx, ctypes.c_void_p(store.ctypes.data),
                                  ctypes.c_void_p(M.fac.addr), store.nbytes), "ocp_d2h")
        out[mc] = (store, M(eng.from_host(v)).to_host())
    np.testing.assert_array_equal(out["1"][0], out["0"][0])
    assert rel_l2(out["1"][1], out["0"][1]) <= 1e-13
