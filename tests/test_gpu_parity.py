"""Parity of the CUDA path (through the C ABI) with the oracle and the golden fixtures.

Tolerances: the local residual is evaluated in the reference's rounding
order, so it is compared bitwise for the polynomial phi's and to 4 ulps
(relative 1e-15 of the row scale) where exp/pow are involved (CUDA vs glibc
libm).  Directions / JVPs come from a no-pivot banded LU instead of SuperLU:
relative 1e-10.  Solves: BASELINE parity bar, y/p/u within 1e-8 relative L2,
iteration counts within +-1.
"""

import numpy as np
import pytest

import raspen_oracle as O
from conftest import golden
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
    if "y" in g.files:
        assert rel_l2(y, g["y"]) <= 1e-8
        assert rel_l2(p, g["p"]) <= 1e-8
        assert rel_l2(u, g["u"]) <= 1e-8
        support_ref = np.abs(g["p"]) > cfg.mu
        support = np.abs(p) > cfg.mu
        band = np.abs(np.abs(g["p"]) - cfg.mu) <= cfg.eps_min
        assert np.array_equal(support[~band], support_ref[~band])
    for key, vec in (("y", y), ("p", p), ("u", u)):
        stride = int(g[f"{key}_stride"])
        samples = g[f"{key}_samples"]
        assert rel_l2(vec[::stride], samples) <= 1e-8, key
        assert abs(np.linalg.norm(vec) - float(g[f"{key}_norm"])) <= 1e-8 * float(g[f"{key}_norm"])


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
