"""Single-CTA vs multi-CTA (k_block_factor_mc) factor of wide subdomains:
bitwise-identical solves, wall time (OCP_FACTOR_MC=0 disables the mc path;
run as two processes: python tools/wide_mc_ab.py out.npy)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import (ContinuationSchedule, KrylovConfig, NewtonConfig,  # noqa: E402
                                   build_local_systems, decompose, newton_continuation, raspen_solve)
from paper_2411_00546_b200.linear_ras import GlobalJacobian, global_residual  # noqa: E402
from paper_2411_00546_b200.problems import EXTRA_CONFIGS, BaselineConfig, build_spec  # noqa: E402

out = {}
cfg = EXTRA_CONFIGS["wide2x2"]
spec = build_spec(cfg, with_matrix=False)
dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
eng = build_local_systems(dec, spec)
for r in range(2):
    eng.set_profiling(True)
    eng.reset_stats()
    t0 = time.perf_counter()
    x, rep = raspen_solve(np.zeros(cfg.unknowns), dec, spec, ContinuationSchedule(1.0, 0.1, 1e-6),
                          cfg=NewtonConfig(tol=1e-10), krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000),
                          inner_tol=1e-8)
    st = eng.stats()
    print(f"wide2x2: {time.perf_counter() - t0:.3f} s outer={rep.outer_iters} gmres={rep.gmres_iters} "
          f"factor {st['factor_ms']:.1f} ms jvp {st['jvp_ms']:.1f} ms", flush=True)
out["wide2x2"] = x
for n, s in ((450, 2), (450, 3)):
    c = BaselineConfig(f"n{n}_{s}", n, "cubic", 1e-3, 1e-2, s, s, 2, 1.0, 0.1, 1e-6, "zero", "bumps", bumps=8)
    sp = build_spec(c, with_matrix=False)
    dc = decompose(sp.grid, s, s, 2)
    t0 = time.perf_counter()
    x, rep = raspen_solve(np.zeros(c.unknowns), dc, sp, ContinuationSchedule(1.0, 0.1, 1e-6),
                          cfg=NewtonConfig(tol=1e-10), krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000),
                          inner_tol=1e-7)
    print(f"N={n} {s}x{s} (inner tol 1e-7): {time.perf_counter() - t0:.3f} s conv={rep.converged} "
          f"outer={rep.outer_iters} inner={rep.inner_iters} gmres={rep.gmres_iters}", flush=True)
    out[f"n{n}_{s}"] = x
c = EXTRA_CONFIGS["mono150"]
sp = build_spec(c, with_matrix=False)
e = build_local_systems(decompose(sp.grid, 1, 1, 0), sp)
t0 = time.perf_counter()
x, rep = newton_continuation(e.from_host(np.zeros(c.unknowns)), lambda x, ep: global_residual(e, x, ep),
                             lambda x, ep: GlobalJacobian(e, x, ep), ContinuationSchedule(1.0, 0.1, 1e-6),
                             NewtonConfig(tol=1e-10, linear_solver="direct"))
print(f"mono150 direct: {time.perf_counter() - t0:.3f} s outer={rep.outer_iters}", flush=True)
out["mono150"] = x.to_host()
np.savez(sys.argv[1], **out)
