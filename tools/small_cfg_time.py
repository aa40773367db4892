"""Wall time and kernel split of the small BASELINE configs 1 and 2 (latency-bound solves)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2411_00546_b200 import ContinuationSchedule, KrylovConfig, NewtonConfig, decompose, raspen_solve, build_local_systems
from paper_2411_00546_b200.problems import CONFIGS, build_spec
import cProfile, pstats
for name in ("cfg1", "cfg2"):
    cfg = CONFIGS[name]
    spec = build_spec(cfg, with_matrix=False)
    dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
    eng = build_local_systems(dec, spec)
    for r in range(3):
        eng.set_profiling(True); eng.reset_stats()
        t0 = time.perf_counter()
        x, rep = raspen_solve(np.zeros(cfg.unknowns), dec, spec, ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min), cfg=NewtonConfig(tol=1e-10), krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000), inner_tol=1e-8)
        wall = time.perf_counter() - t0
        st = eng.stats()
    print(name, f"{wall*1e3:.1f} ms", {k: round(v, 2) for k, v in st.items() if k.endswith('_ms') or k=='launches'}, flush=True)
    pr = cProfile.Profile(); pr.enable()
    x, rep = raspen_solve(np.zeros(cfg.unknowns), dec, spec, ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min), cfg=NewtonConfig(tol=1e-10), krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000), inner_tol=1e-8)
    pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(8)
