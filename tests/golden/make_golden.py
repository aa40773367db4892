"""Generate golden fixtures by running the UNMODIFIED reference package.

Runs only in the build container, where the reference is importable from
``/root/reference/pkg/src`` (read-only).  The GPU box never runs this file;
it only reads the ``.npz`` files written here.

Usage::

    python tests/golden/make_golden.py cfg1 [--inner-tol 1e-8] [--threads 8]
    python tests/golden/make_golden.py cfg5 --threads 8        # sweep + JVP
    python tests/golden/make_golden.py units                   # small unit fixtures
    python tests/golden/make_golden.py ras_units               # linear-RAS operator fixtures
    python tests/golden/make_golden.py ras_cfg1                # newton-ras-eps solve

Settings are the harness-equivalent ones of SURVEY.md 0.10: outer tol 1e-10,
GMRES rel 1e-8 / max 1000 (`harness/experiments.py:63-70`), inner tol as given
(1e-8 reference default; 1e-7 is the documented deviation for configs 3-4),
inner max_outer 200, sigma 1.1 / 30 halvings, continuation on.

Inputs come from ``paper_2411_00546_b200.problems`` (plain numpy, no GPU);
the phi objects are duck-typed into the reference's ``ProblemSpec``
(SURVEY.md 0.3).
"""

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import ocp.schwarz as ref_schwarz  # noqa: E402
from ocp.grid import Grid as RefGrid, build_laplacian as ref_laplacian  # noqa: E402
from ocp.krylov import KrylovConfig  # noqa: E402
from ocp.newton import ContinuationSchedule, NewtonConfig  # noqa: E402
from ocp.system import ProblemSpec as RefSpec, recover_control  # noqa: E402

from paper_2411_00546_b200.problems import CONFIGS, build_fields  # noqa: E402
from paper_2411_00546_b200.system import make_phi, Nonlinearity  # noqa: E402

DIGEST_SEED = 20241101
DIGEST_PROJ = 16
DIGEST_SAMPLES = 16384


def digest(v):
    """Size-independent summary of a long field (norms, samples, projections)."""
    v = np.asarray(v, dtype=float)
    stride = max(1, v.shape[0] // DIGEST_SAMPLES)
    rng = np.random.default_rng(DIGEST_SEED + v.shape[0])
    signs = rng.integers(0, 2, size=(DIGEST_PROJ, v.shape[0])).astype(np.float64) * 2.0 - 1.0
    return {
        "norm": float(np.linalg.norm(v)),
        "stride": stride,
        "samples": v[::stride].copy(),
        "proj": signs @ v,
    }


def support_bits(p, mu, eps):
    """Full-grid control support of the reference solution, bit-packed.

    `supp_bits`: |p| > mu, i.e. u != 0 of the unsmoothed projection
    (`system.py:173-174` at eps -> 0); `band_bits`: ||p| - mu| <= eps, the
    points where the north-star support criterion is waived.  One bit per
    grid point, so the whole 1023^2 grid fits in ~2 x 131 KB before
    compression.
    """
    p = np.asarray(p, dtype=float)
    return {
        "supp_bits": np.packbits(np.abs(p) > mu),
        "band_bits": np.packbits(np.abs(np.abs(p) - mu) <= eps),
        "supp_count": int(np.count_nonzero(np.abs(p) > mu)),
    }


def ref_spec(cfg):
    grid = RefGrid(cfg.n)
    f, y_d = build_fields(cfg)
    return RefSpec(grid=grid, a=ref_laplacian(grid), phi=make_phi(cfg.phi),
                   nu=cfg.nu, mu=cfg.mu, f=f, y_d=y_d)


class PerSubRecorder:
    """Wraps schwarz._solve_local to record per-subdomain inner counts."""

    def __init__(self):
        self.calls = []
        self._orig = ref_schwarz._solve_local

    def __enter__(self):
        rec = self.calls
        orig = self._orig

        def wrapped(i, sub, loc, spec, x, sched, cfg):
            v, k = orig(i, sub, loc, spec, x, sched, cfg)
            rec.append((i, k))
            return v, k

        ref_schwarz._solve_local = wrapped
        return self

    def __exit__(self, *exc):
        ref_schwarz._solve_local = self._orig

    def per_eval(self, n_sub):
        out = []
        for start in range(0, len(self.calls) - n_sub + 1, n_sub):
            chunk = dict(self.calls[start:start + n_sub])
            if len(chunk) == n_sub:
                out.append([chunk[i] for i in range(n_sub)])
        return out


def run_solve(name, inner_tol, threads, out_path):
    cfg = CONFIGS[name]
    spec = ref_spec(cfg)
    dec = ref_schwarz.decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    sched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)
    x0 = np.zeros(2 * spec.grid.size)
    t0 = time.perf_counter()
    with PerSubRecorder() as rec:
        x, report = ref_schwarz.raspen_solve(
            x0, dec, spec, sched,
            cfg=NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1),
            krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000),
            inner_tol=inner_tol, threads=threads, continuation=True)
    wall = time.perf_counter() - t0
    n2 = spec.grid.size
    y, p = x[:n2], x[n2:]
    u = recover_control(p, spec, cfg.eps_min)
    data = dict(
        config=name, inner_tol=inner_tol, threads=threads, wall=wall,
        converged=report.converged, outer_iters=report.outer_iters,
        residual_norms=np.array(report.residual_norms),
        eps_values=np.array(report.eps_values),
        alphas=np.array(report.alphas),
        gmres_iters=np.array([-1 if k is None else k for k in report.gmres_iters]),
        inner_iters=np.array(report.inner_iters),
        threshold=report.threshold,
        failure="" if report.failure is None else report.failure,
        per_sub=np.array(rec.per_eval(len(dec)), dtype=np.int64),
        n_calls=len(rec.calls),
    )
    if n2 <= 256 * 256:
        data.update(y=y, p=p, u=u)
    for key, vec in (("y", y), ("p", p), ("u", u)):
        for k, v in digest(vec).items():
            data[f"{key}_{k}"] = v
    data.update(support_bits(p, cfg.mu, cfg.eps_min))
    np.savez_compressed(out_path, **data)
    print(f"{name} inner_tol={inner_tol}: converged={report.converged} "
          f"outer={report.outer_iters} inner={report.inner_iters} "
          f"gmres={report.gmres_iters} failure={report.failure} wall={wall:.1f}s")


def run_sweep(name, threads, out_path):
    """Config 5: one RAS sweep at x = 0 (eps fixed) plus one JVP."""
    cfg = CONFIGS[name]
    spec = ref_spec(cfg)
    dec = ref_schwarz.decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    x = np.zeros(2 * spec.grid.size)
    eps = cfg.eps_min
    t0 = time.perf_counter()
    with PerSubRecorder() as rec:
        f_val, corr = ref_schwarz.raspen_residual(
            x, dec, spec, eps, inner_cfg=NewtonConfig(tol=1e-8, max_outer=200),
            inner_sched=ContinuationSchedule.fixed(eps), threads=threads)
    t1 = time.perf_counter()
    d = np.random.default_rng(1).standard_normal(x.shape[0])
    out = ref_schwarz.raspen_jacobian_apply(x, d, dec, spec, eps, corr)
    t2 = time.perf_counter()
    data = dict(config=name, threads=threads, sweep_wall=t1 - t0, jvp_wall=t2 - t1,
                inner_iters=np.array(corr.inner_iters, dtype=np.int64))
    for key, vec in (("fval", f_val), ("jvp", out)):
        for k, v in digest(vec).items():
            data[f"{key}_{k}"] = v
    np.savez_compressed(out_path, **data)
    print(f"{name}: sweep {t1 - t0:.1f}s jvp {t2 - t1:.2f}s inner={set(corr.inner_iters)}")


def run_units(out_path):
    """Small fixtures that pin individual operators of the reference.

    * local residuals of every subdomain at a random x (`schwarz.py:174-186`),
    * one raspen_residual + JVP at a random iterate (`schwarz.py:285-345`),
    * full raspen_solve on the kappa family (`schwarz.py:348-411`),
    for both the kappa family and the cubic / expm1 duck-typed phis.
    """
    from paper_2411_00546_b200.problems import mild_spec

    data = {}
    cases = [
        ("kappa16", 16, 2, 2, 2, Nonlinearity(0.1), 1e-2, 1.0),
        ("cubic20", 20, 2, 3, 2, make_phi("cubic"), 1e-3, 1e-2),
        ("expm1_18", 18, 3, 2, 3, make_phi("expm1"), 1e-4, 5e-3),
    ]
    for tag, n, s1, s2, m, phi, nu, mu in cases:
        base = mild_spec(n)
        grid = RefGrid(n)
        spec = RefSpec(grid=grid, a=ref_laplacian(grid), phi=phi, nu=nu, mu=mu,
                       f=base.f, y_d=10.0 * base.y_d)
        dec = ref_schwarz.decompose(grid, s1, s2, m)
        systems = ref_schwarz.build_local_systems(dec, spec)
        rng = np.random.default_rng(100 + n)
        x = 0.3 * rng.standard_normal(2 * grid.size)
        eps = 1e-2
        loc_res = []
        for sub, loc in zip(dec.subdomains, systems):
            res, _ = ref_schwarz._local_problem(loc, spec, x)
            loc_res.append(res(x[sub.pair_idx] + 0.01, eps))
        data[f"{tag}_x"] = x
        data[f"{tag}_local_res"] = np.concatenate(loc_res)
        f_val, corr = ref_schwarz.raspen_residual(
            x, dec, spec, eps, inner_cfg=NewtonConfig(tol=1e-10), threads=1)
        d = rng.standard_normal(x.shape[0])
        data[f"{tag}_fval"] = f_val
        data[f"{tag}_inner"] = np.array(corr.inner_iters)
        data[f"{tag}_d"] = d
        data[f"{tag}_jvp"] = ref_schwarz.raspen_jacobian_apply(x, d, dec, spec, eps, corr)
        sched = ContinuationSchedule(1.0, 0.2, 1e-3)
        with PerSubRecorder() as rec:
            xs, rep = ref_schwarz.raspen_solve(
                np.zeros_like(x), dec, spec, sched,
                cfg=NewtonConfig(tol=1e-10),
                krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000), threads=1)
        data[f"{tag}_solve_x"] = xs
        data[f"{tag}_solve_converged"] = rep.converged
        data[f"{tag}_solve_outer"] = rep.outer_iters
        data[f"{tag}_solve_inner"] = np.array(rep.inner_iters)
        data[f"{tag}_solve_gmres"] = np.array(rep.gmres_iters)
        data[f"{tag}_solve_norms"] = np.array(rep.residual_norms)
        data[f"{tag}_solve_per_sub"] = np.array(rec.per_eval(len(dec)))
        print(f"{tag}: inner={corr.inner_iters} solve outer={rep.outer_iters} "
              f"inner={rep.inner_iters} gmres={rep.gmres_iters} conv={rep.converged}")
    np.savez_compressed(out_path, **data)


def run_variants(out_path):
    """Reference behaviour off the harness defaults (`schwarz.py:211-218,285-324,348-411`).

    * ``raspen_solve(continuation=False)`` (`pkg/tests/test_schwarz.py:350-358`)
      and ``raspen_solve(backtracking=True)`` (sigma 1.1 outer line search) on
      the unit cases and on BASELINE config 1;
    * ``raspen_residual`` with an inner schedule whose floor differs from eps
      (solve with the schedule, refactor at eps: `schwarz.py:296-315`) and the
      JVP from those stored factors;
    * ``local_correction(i)`` of single subdomains (`schwarz.py:211-218`).
    """
    from paper_2411_00546_b200.problems import mild_spec

    data = {}
    cases = [
        ("kappa16", 16, 2, 2, 2, Nonlinearity(0.1), 1e-2, 1.0),
        ("cubic20", 20, 2, 3, 2, make_phi("cubic"), 1e-3, 1e-2),
    ]
    specs = []
    for tag, n, s1, s2, m, phi, nu, mu in cases:
        base = mild_spec(n)
        grid = RefGrid(n)
        spec = RefSpec(grid=grid, a=ref_laplacian(grid), phi=phi, nu=nu, mu=mu,
                       f=base.f, y_d=10.0 * base.y_d)
        specs.append((tag, spec, ref_schwarz.decompose(grid, s1, s2, m),
                      ContinuationSchedule(1.0, 0.2, 1e-3)))
    cfg = CONFIGS["cfg1"]
    spec1 = ref_spec(cfg)
    specs.append(("cfg1", spec1, ref_schwarz.decompose(spec1.grid, cfg.s1, cfg.s2, cfg.overlap),
                  ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)))
    for tag, spec, dec, sched in specs:
        x0 = np.zeros(2 * spec.grid.size)
        for var, kw in (("nocont", dict(continuation=False)),
                        ("backtrack", dict(backtracking=True))):
            with PerSubRecorder() as rec:
                xs, rep = ref_schwarz.raspen_solve(
                    x0, dec, spec, sched, cfg=NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1),
                    krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000), threads=1, **kw)
            k = f"{tag}_{var}"
            data[f"{k}_x"] = xs
            data[f"{k}_converged"] = rep.converged
            data[f"{k}_outer"] = rep.outer_iters
            data[f"{k}_inner"] = np.array(rep.inner_iters)
            data[f"{k}_gmres"] = np.array([-1 if g is None else g for g in rep.gmres_iters])
            data[f"{k}_norms"] = np.array(rep.residual_norms)
            data[f"{k}_alphas"] = np.array(rep.alphas)
            data[f"{k}_per_sub"] = np.array(rec.per_eval(len(dec)))
            print(f"{k}: conv={rep.converged} outer={rep.outer_iters} inner={rep.inner_iters} "
                  f"gmres={rep.gmres_iters} alphas={rep.alphas}")
        if tag == "cfg1":
            continue
        rng = np.random.default_rng(300 + spec.grid.n)
        x = 0.3 * rng.standard_normal(2 * spec.grid.size)
        d = rng.standard_normal(x.shape[0])
        eps = 1e-2
        # inner continuation to a floor below eps, then refactorisation at eps
        f_val, corr = ref_schwarz.raspen_residual(
            x, dec, spec, eps, inner_cfg=NewtonConfig(tol=1e-10),
            inner_sched=ContinuationSchedule(1.0, 0.2, 1e-3), threads=1)
        data[f"{tag}_floor_x"] = x
        data[f"{tag}_floor_d"] = d
        data[f"{tag}_floor_fval"] = f_val
        data[f"{tag}_floor_inner"] = np.array(corr.inner_iters)
        data[f"{tag}_floor_jvp"] = ref_schwarz.raspen_jacobian_apply(x, d, dec, spec, eps, corr)
        for i in (0, len(dec) - 1):
            data[f"{tag}_lc{i}"] = ref_schwarz.local_correction(
                i, x, dec, spec, eps, inner_cfg=NewtonConfig(tol=1e-10))
        print(f"{tag}: floor inner={corr.inner_iters}")
    np.savez_compressed(out_path, **data)


def _ras_solve_args(spec, dec, gmres_tol=1e-8, tol=1e-10, sigma=1.1, max_outer=200):
    """The `newton-ras-eps` branch of `solve_single` (`harness/experiments.py:72-84`)."""
    from ocp.system import residual, jacobian

    systems = ref_schwarz.build_local_systems(dec, spec)
    newton_cfg = NewtonConfig(tol=tol, max_outer=max_outer, sigma=sigma,
                              linear_solver=KrylovConfig(rel_tol=gmres_tol, max_iters=2000))
    return (lambda x, eps: residual(x, spec, eps, check=False),
            lambda x, eps: jacobian(x, spec, eps),
            newton_cfg,
            lambda x, eps: ref_schwarz.ras_preconditioner(x, dec, spec, eps, systems))


def run_ras_units(out_path):
    """Global residual / Jacobian action and one RAS preconditioner application
    (`system.py:147-160`, `schwarz.py:221-239`), plus a small full solve."""
    from ocp.newton import newton_continuation
    from ocp.system import residual, jacobian
    from paper_2411_00546_b200.problems import mild_spec

    data = {}
    cases = [
        ("cubic20", 20, 2, 3, 2, make_phi("cubic"), 1e-3, 1e-2),
        ("expm1_18", 18, 3, 2, 3, make_phi("expm1"), 1e-4, 5e-3),
        ("kappa16", 16, 2, 2, 2, Nonlinearity(0.1), 1e-2, 1.0),
    ]
    for tag, n, s1, s2, m, phi, nu, mu in cases:
        base = mild_spec(n)
        grid = RefGrid(n)
        spec = RefSpec(grid=grid, a=ref_laplacian(grid), phi=phi, nu=nu, mu=mu,
                       f=base.f, y_d=10.0 * base.y_d)
        dec = ref_schwarz.decompose(grid, s1, s2, m)
        rng = np.random.default_rng(200 + n)
        x = 0.3 * rng.standard_normal(2 * grid.size)
        d = rng.standard_normal(2 * grid.size)
        eps = 1e-2
        data[f"{tag}_x"] = x
        data[f"{tag}_d"] = d
        data[f"{tag}_resid"] = residual(x, spec, eps, check=False)
        data[f"{tag}_jvp"] = jacobian(x, spec, eps) @ d
        data[f"{tag}_prec"] = ref_schwarz.ras_precondition(d, x, dec, spec, eps)
        res_fn, jac_fn, ncfg, pb = _ras_solve_args(spec, dec)
        xs, rep = newton_continuation(np.zeros_like(x), res_fn, jac_fn,
                                      ContinuationSchedule(1.0, 0.2, 1e-3), ncfg,
                                      precond_builder=pb)
        data[f"{tag}_solve_x"] = xs
        data[f"{tag}_solve_converged"] = rep.converged
        data[f"{tag}_solve_outer"] = rep.outer_iters
        data[f"{tag}_solve_gmres"] = np.array(rep.gmres_iters)
        data[f"{tag}_solve_norms"] = np.array(rep.residual_norms)
        data[f"{tag}_solve_alphas"] = np.array(rep.alphas)
        print(f"{tag}: ras solve outer={rep.outer_iters} gmres={rep.gmres_iters} "
              f"alphas={rep.alphas} conv={rep.converged}")
    np.savez_compressed(out_path, **data)


def run_ras_solve(name, out_path):
    """`newton-ras-eps` on a BASELINE configuration (harness settings)."""
    from ocp.newton import newton_continuation

    cfg = CONFIGS[name]
    spec = ref_spec(cfg)
    dec = ref_schwarz.decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    sched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)
    res_fn, jac_fn, ncfg, pb = _ras_solve_args(spec, dec)
    t0 = time.perf_counter()
    x, report = newton_continuation(np.zeros(2 * spec.grid.size), res_fn, jac_fn, sched, ncfg,
                                    precond_builder=pb)
    wall = time.perf_counter() - t0
    n2 = spec.grid.size
    y, p = x[:n2], x[n2:]
    u = recover_control(p, spec, cfg.eps_min)
    data = dict(
        config=name, method="newton-ras-eps", wall=wall,
        converged=report.converged, outer_iters=report.outer_iters,
        residual_norms=np.array(report.residual_norms),
        eps_values=np.array(report.eps_values),
        alphas=np.array(report.alphas),
        gmres_iters=np.array([-1 if k is None else k for k in report.gmres_iters]),
        threshold=report.threshold,
        failure="" if report.failure is None else report.failure,
    )
    if n2 <= 256 * 256:
        data.update(y=y, p=p, u=u)
    for key, vec in (("y", y), ("p", p), ("u", u)):
        for k, v in digest(vec).items():
            data[f"{key}_{k}"] = v
    data.update(support_bits(p, cfg.mu, cfg.eps_min))
    np.savez_compressed(out_path, **data)
    print(f"ras {name}: converged={report.converged} outer={report.outer_iters} "
          f"gmres={report.gmres_iters} alphas={report.alphas} failure={report.failure} "
          f"wall={wall:.1f}s")


def run_wide(out_path):
    """Decompositions beyond the fast kernels' 112-point short side.

    * ``wide2x2``: raspen_solve on a 300^2 grid, 2x2 subdomains, overlap 8
      (local short side 158; harness settings, inner tol 1e-8);
    * ``mono150``: monolithic newton-eps with the direct (SuperLU) direction
      on a 150^2 grid (`harness/experiments.py:86-91`), i.e. one banded
      solve of the whole 2 x 22500-unknown Jacobian per Newton step.
    """
    from ocp.newton import newton_continuation
    from ocp.system import residual, jacobian
    from paper_2411_00546_b200.problems import EXTRA_CONFIGS

    data = {}
    cfg = EXTRA_CONFIGS["wide2x2"]
    spec = ref_spec(cfg)
    dec = ref_schwarz.decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    sched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)
    t0 = time.perf_counter()
    with PerSubRecorder() as rec:
        x, rep = ref_schwarz.raspen_solve(
            np.zeros(2 * spec.grid.size), dec, spec, sched,
            cfg=NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1),
            krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000), inner_tol=1e-8, threads=4)
    print(f"wide2x2: conv={rep.converged} outer={rep.outer_iters} inner={rep.inner_iters} "
          f"gmres={rep.gmres_iters} wall={time.perf_counter() - t0:.1f}s", flush=True)
    _store_solve(data, "wide2x2", cfg, spec, x, rep)
    data["wide2x2_per_sub"] = np.array(rec.per_eval(len(dec)), dtype=np.int64)

    cfg = EXTRA_CONFIGS["mono150"]
    spec = ref_spec(cfg)
    sched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)
    t0 = time.perf_counter()
    x, rep = newton_continuation(np.zeros(2 * spec.grid.size),
                                 lambda x, eps: residual(x, spec, eps, check=False),
                                 lambda x, eps: jacobian(x, spec, eps), sched,
                                 NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1,
                                              linear_solver="direct"))
    print(f"mono150: conv={rep.converged} outer={rep.outer_iters} alphas={rep.alphas} "
          f"wall={time.perf_counter() - t0:.1f}s", flush=True)
    _store_solve(data, "mono150", cfg, spec, x, rep)
    np.savez_compressed(out_path, **data)


def _store_solve(data, tag, cfg, spec, x, rep):
    n2 = spec.grid.size
    y, p = x[:n2], x[n2:]
    u = recover_control(p, spec, cfg.eps_min)
    data[f"{tag}_converged"] = rep.converged
    data[f"{tag}_outer"] = rep.outer_iters
    data[f"{tag}_inner"] = np.array(rep.inner_iters)
    data[f"{tag}_gmres"] = np.array([-1 if k is None else k for k in rep.gmres_iters])
    data[f"{tag}_alphas"] = np.array(rep.alphas)
    data[f"{tag}_norms"] = np.array(rep.residual_norms)
    for key, vec in (("y", y), ("p", p), ("u", u)):
        for k, v in digest(vec).items():
            data[f"{tag}_{key}_{k}"] = v
    for k, v in support_bits(p, cfg.mu, cfg.eps_min).items():
        data[f"{tag}_{k}"] = v


HARNESS_CASES = [
    ("newton_eps", dict(method="newton-eps")),
    ("newton", dict(method="newton", eps0=1e-3)),
    ("newton_eps_gmres", dict(method="newton-eps", linear_solver="gmres")),
    ("newton_ras_eps", dict(method="newton-ras-eps", s1=2, s2=2, overlap=2)),
    ("raspen_eps", dict(method="raspen-eps", s1=2, s2=2, overlap=2)),
    ("raspen_eps_23", dict(method="raspen-eps", n=20, s1=2, s2=3, overlap=1, k_tilde=3)),
    ("fail_max_outer", dict(method="newton-eps", max_outer=1, eps_min=1e-10)),
]
HARNESS_MILD = dict(n=12, nu=1e-2, k_tilde=2, eps_min=1e-3)   # pkg/tests/test_harness.py:27


def run_harness(out_path):
    """Artifacts of the reference's run_single (`harness/experiments.py:102-117`)
    on the mild configuration family of its own tests, plus manufactured
    problems (`system.py:219-265`)."""
    import tempfile
    from pathlib import Path
    from ocp.harness.config import build_config
    from ocp.harness.experiments import run_single
    from ocp.system import construct_plateau_problem, construct_test_problem

    data = {}
    for tag, over in HARNESS_CASES:
        cfg = build_config(overrides={**HARNESS_MILD, **over})
        with tempfile.TemporaryDirectory() as tmp:
            code, rep = run_single(cfg, tmp)
            for name in ("report.json", "residual_history.csv", "y.csv", "p.csv", "u.csv"):
                data[f"{tag}__{name}"] = np.array((Path(tmp) / name).read_text())
        data[f"{tag}__code"] = code
        print(f"harness {tag}: code={code} outer={rep['outer_iters']} gmres={rep['gmres_iters']}")
    for tag, n, kw in (("test12", 12, dict(kappa=0.1, nu=1e-2, mu=1.0, k_tilde=2)),
                       ("test40", 40, dict(kappa=0.1, nu=1e-6, mu=1.0, k_tilde=5))):
        spec, pair = construct_test_problem(RefGrid(n), **kw)
        data[f"mfg_{tag}_yd"], data[f"mfg_{tag}_y"], data[f"mfg_{tag}_p"] = spec.y_d, pair.y, pair.p
    spec, pair = construct_plateau_problem(RefGrid(24), kappa=0.1, nu=1e-3, mu=1.0)
    data["mfg_plateau24_yd"], data["mfg_plateau24_y"], data["mfg_plateau24_p"] = \
        spec.y_d, pair.y, pair.p
    np.savez_compressed(out_path, **data)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what")
    ap.add_argument("--inner-tol", type=float, default=1e-8)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if args.what == "units":
        run_units(args.out or os.path.join(HERE, "units.npz"))
    elif args.what == "harness":
        run_harness(args.out or os.path.join(HERE, "harness.npz"))
    elif args.what == "wide":
        run_wide(args.out or os.path.join(HERE, "wide.npz"))
    elif args.what == "variants":
        run_variants(args.out or os.path.join(HERE, "variants.npz"))
    elif args.what == "ras_units":
        run_ras_units(args.out or os.path.join(HERE, "ras_units.npz"))
    elif args.what.startswith("ras_cfg"):
        run_ras_solve(args.what[4:], args.out or os.path.join(HERE, f"{args.what}.npz"))
    elif args.what.startswith("cfg5"):
        run_sweep(args.what, args.threads, args.out or os.path.join(HERE, f"{args.what}_sweep.npz"))
    else:
        tag = f"{args.what}_tol{args.inner_tol:g}"
        run_solve(args.what, args.inner_tol, args.threads,
                  args.out or os.path.join(HERE, f"{tag}.npz"))


if __name__ == "__main__":
    main()
