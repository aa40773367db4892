"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck, one tool per process):

* RASPEN solve on the cubic20 unit case and BASELINE config 1 - local
  residual (tickets), batched block factor (12-warp and narrow instances),
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
