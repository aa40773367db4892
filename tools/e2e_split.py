"""Where the end-to-end raspen_solve time goes beyond the device solve (config 4):
engine (context) build with a fresh ProblemSpec, x0 upload, solve, x download."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import KrylovConfig, NewtonConfig, build_local_systems, raspen_solve  # noqa: E402
from paper_2411_00546_b200.problems import CONFIGS  # noqa: E402
from paper_2411_00546_b200.system import ProblemSpec  # noqa: E402

sys.argv = ["bench.py"]
import bench  # noqa: E402

cfg, spec, dec, sched = bench.problem()
newton_cfg = NewtonConfig(tol=1e-10, max_outer=200, sigma=1.1)
kry = KrylovConfig(rel_tol=1e-8, max_iters=1000)
x0 = np.zeros(cfg.unknowns)
for rep in range(4):
    fresh = ProblemSpec(grid=spec.grid, a=None, phi=spec.phi, nu=spec.nu, mu=spec.mu,
                        f=spec.f.copy(), y_d=spec.y_d.copy())
    t0 = time.perf_counter()
    eng = build_local_systems(dec, fresh)
    t1 = time.perf_counter()
    x, r = raspen_solve(x0, dec, fresh, sched, cfg=newton_cfg, krylov_cfg=kry, inner_tol=1e-7)
    t2 = time.perf_counter()
    print(f"build {1e3 * (t1 - t0):.1f} ms, solve+io {1e3 * (t2 - t1):.1f} ms, conv {r.converged}")
    dec.__dict__.get("_engines", {}).pop(id(fresh), None)
    del fresh, eng
