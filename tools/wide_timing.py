"""Wall time of coarse decompositions on the wide-line kernels: the paper's
N = 450 problem sizes (2x2, 3x3, 4x4 RASPEN) with the
config-2 style data, and monolithic direct Newton on n = 150 / 300 / 450."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import (ContinuationSchedule, KrylovConfig, NewtonConfig,  # noqa: E402
                                   build_local_systems, decompose, newton_continuation, raspen_solve)
from paper_2411_00546_b200.linear_ras import GlobalJacobian, global_residual  # noqa: E402
from paper_2411_00546_b200.problems import BaselineConfig, build_spec  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
for s in ((2, 3, 4) if which in ("all", "raspen") else ()) if which != "raspen1" else (2,):
    cfg = BaselineConfig(f"n450_{s}x{s}", 450, "cubic", 1e-3, 1e-2, s, s, 2, 1.0, 0.1, 1e-6,
                         "zero", "bumps", bumps=8)
    spec = build_spec(cfg, with_matrix=False)
    dec = decompose(spec.grid, s, s, 2)
    for rep_i in range(1 if which == "raspen1" else 2):
        t0 = time.perf_counter()
        x, rep = raspen_solve(np.zeros(cfg.unknowns), dec, spec, ContinuationSchedule(1.0, 0.1, 1e-6),
                              cfg=NewtonConfig(tol=1e-10), krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000),
                              inner_tol=1e-8)
        print(f"RASPEN N=450 {s}x{s} overlap 2: {time.perf_counter() - t0:.3f} s conv={rep.converged} "
              f"outer={rep.outer_iters} inner={rep.inner_iters} gmres={rep.gmres_iters}", flush=True)
for n in ((150, 300, 450) if which in ("all", "mono") else (int(which[4:]),) if which.startswith("mono") and which[4:] else ()):
    cfg = BaselineConfig(f"mono{n}", n, "cubic", 1e-3, 1e-2, 1, 1, 0, 1.0, 0.1, 1e-6, "zero", "bumps", bumps=8)
    spec = build_spec(cfg, with_matrix=False)
    eng = build_local_systems(decompose(spec.grid, 1, 1, 0), spec)
    t0 = time.perf_counter()
    x, rep = newton_continuation(eng.from_host(np.zeros(cfg.unknowns)), lambda x, e: global_residual(eng, x, e),
                                 lambda x, e: GlobalJacobian(eng, x, e), ContinuationSchedule(1.0, 0.1, 1e-6),
                                 NewtonConfig(tol=1e-10, linear_solver="direct"))
    print(f"monolithic direct n={n}: {time.perf_counter() - t0:.3f} s conv={rep.converged} "
          f"outer={rep.outer_iters}", flush=True)
