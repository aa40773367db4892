"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck, one tool per process):

* RASPEN solve on the cubic20 unit case and BASELINE config 1 - local
  residual (per-CTA partials), batched block factor (12-warp and narrow instances),
  block solve (mbarrier TMA ring, named barriers), fused JVP, cooperative
  lagged-dot Arnoldi (atomic grid barrier), scatter / vector kernels;
* newton-ras-eps on config 1 - global residual / Jacobian / JVP, RAS apply;
* device state solve (CG) of a manufactured problem.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_00546_b200 import (ContinuationSchedule, Grid, KrylovConfig, NewtonConfig,  # noqa: E402
                                   ProblemSpec, construct_test_problem, decompose, make_phi,
                                   newton_ras_solve, raspen_solve)
from paper_2411_00546_b200.problems import CONFIGS, build_spec, mild_spec  # noqa: E402

n = 20
base = mild_spec(n)
spec = ProblemSpec(grid=Grid(n), a=None, phi=make_phi("cubic"), nu=1e-3, mu=1e-2, f=base.f,
                   y_d=10.0 * base.y_d)
x, rep = raspen_solve(np.zeros(2 * n * n), decompose(spec.grid, 2, 3, 2), spec,
                      ContinuationSchedule(1.0, 0.2, 1e-3), cfg=NewtonConfig(tol=1e-10),
                      krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000))
print("cubic20 raspen:", rep.converged, rep.outer_iters, rep.gmres_iters, flush=True)

cfg = CONFIGS["cfg1"]
spec1 = build_spec(cfg, with_matrix=False)
dec1 = decompose(spec1.grid, cfg.s1, cfg.s2, cfg.overlap)
sched1 = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min)
x, rep = raspen_solve(np.zeros(cfg.unknowns), dec1, spec1, sched1,
                      cfg=NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1),
                      krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000), inner_tol=1e-8)
print("cfg1 raspen:", rep.converged, rep.outer_iters, rep.gmres_iters, flush=True)

if "--all" in sys.argv:
    spec1m = build_spec(cfg)
    x, rep = newton_ras_solve(np.zeros(cfg.unknowns), dec1, spec1m, sched1,
                              NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1,
                                           linear_solver=KrylovConfig(rel_tol=1e-8, max_iters=2000)))
    print("cfg1 newton-ras:", rep.converged, rep.outer_iters, rep.gmres_iters, flush=True)
    spec_t, pair = construct_test_problem(Grid(12), kappa=0.1, nu=1e-2, mu=1.0, k_tilde=2)
    print("manufactured test12:", float(np.abs(pair.y).max()), flush=True)

if "--big" in sys.argv:   # oversized-block paths: config 4 (n = 172 corner), config 5 (ragged)
    from paper_2411_00546_b200 import build_local_systems
    from paper_2411_00546_b200.schwarz import _jvp, _sweep, release_local_systems
    for name, tol in (("cfg4", 1e-7), ("cfg5", 1e-8)):
        c = CONFIGS[name]
        sp_ = build_spec(c, with_matrix=False)
        dc = decompose(sp_.grid, c.s1, c.s2, c.overlap)
        eng = build_local_systems(dc, sp_)
        xd = eng.from_host(np.zeros(c.unknowns))
        fac = eng.factor_store()
        sch = (ContinuationSchedule(c.eps0, c.gamma, c.eps_min) if name == "cfg4"
               else ContinuationSchedule.fixed(c.eps_min))
        fval, inner = _sweep(eng, xd, fac, sch, NewtonConfig(tol=tol, max_outer=200))
        out = _jvp(eng, fac, eng.from_host(np.random.default_rng(1).standard_normal(c.unknowns)))
        print(f"{name} sweep + JVP: inner max {max(inner)}, |fval| {fval.norm():.6e}, "
              f"|jvp| {out.norm():.6e}", flush=True)
        del out, fval, fac, xd, eng
        release_local_systems(dc)

if "--wide" in sys.argv:   # wide lines: k_block_factor_mc, k_block_solve_mc, k_block_solve_wide
    from paper_2411_00546_b200 import build_local_systems, newton_continuation
    from paper_2411_00546_b200.linear_ras import GlobalJacobian, global_residual
    from paper_2411_00546_b200.problems import EXTRA_CONFIGS
    c = EXTRA_CONFIGS["wide2x2"]
    sp_ = build_spec(c, with_matrix=False)
    dc = decompose(sp_.grid, c.s1, c.s2, c.overlap)
    x, rep = raspen_solve(np.zeros(c.unknowns), dc, sp_, ContinuationSchedule(c.eps0, c.gamma, c.eps_min),
                          cfg=NewtonConfig(tol=1e-10), krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000),
                          inner_tol=1e-8)
    print("wide2x2 raspen:", rep.converged, rep.outer_iters, rep.gmres_iters, flush=True)
    os.environ["OCP_FACTOR_MC"] = "0"   # the single-CTA wide kernels too
    dc2 = decompose(sp_.grid, c.s1, c.s2, c.overlap)
    x2, rep2 = raspen_solve(np.zeros(c.unknowns), dc2, sp_, ContinuationSchedule(c.eps0, c.gamma, c.eps_min),
                            cfg=NewtonConfig(tol=1e-10), krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000),
                            inner_tol=1e-8)
    print("wide2x2 raspen (single-CTA wide kernels):", rep2.converged, rep2.outer_iters, flush=True)
    del os.environ["OCP_FACTOR_MC"]
    c = EXTRA_CONFIGS["mono150"]
    sp_ = build_spec(c, with_matrix=False)
    e = build_local_systems(decompose(sp_.grid, 1, 1, 0), sp_)
    x, rep = newton_continuation(e.from_host(np.zeros(c.unknowns)), lambda x, ep: global_residual(e, x, ep),
                                 lambda x, ep: GlobalJacobian(e, x, ep), ContinuationSchedule(1.0, 0.1, 1e-6),
                                 NewtonConfig(tol=1e-10, linear_solver="direct"))
    print("mono150 direct:", rep.converged, rep.outer_iters, flush=True)

# racecheck stand-in: the same solves repeated must be bitwise identical
# (mbarrier rings, named barriers, grid barrier and tickets all feed
# fixed-order reductions, so any race shows up as a changed bit)
reps = int(os.environ.get("OCP_REPEAT", "0"))
if reps:
    ref = None
    for r in range(reps):
        x, rep = raspen_solve(np.zeros(cfg.unknowns), dec1, spec1, sched1,
                              cfg=NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1),
                              krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000),
                              inner_tol=1e-8)
        key = (x.tobytes(), tuple(rep.gmres_iters), tuple(rep.residual_norms))
        assert ref is None or key == ref, f"repeat {r} differs"
        ref = key
    print(f"{reps} repeated config-1 solves bitwise identical", flush=True)

if os.environ.get("OCP_GUARD") == "1":
    import ctypes
    import gc
    from paper_2411_00546_b200 import _native as nat
    from paper_2411_00546_b200.schwarz import release_local_systems
    release_local_systems(dec1)
    gc.collect()
    lib = nat.load()
    bad, bufs = ctypes.c_longlong(), ctypes.c_longlong()
    rc = lib.ocp_check_guards(ctypes.byref(bad), ctypes.byref(bufs))
    print(f"guard zones: rc={rc} corrupted_bytes={bad.value} live_buffers={bufs.value} "
          f"{nat.last_error(None) if bad.value else ''}", flush=True)
    sys.exit(1 if rc or bad.value else 0)
