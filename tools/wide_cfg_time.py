"""Wall time and kernel split of the wide2x2 decomposition (300^2, 2x2: local short side 158)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2411_00546_b200 import ContinuationSchedule, KrylovConfig, NewtonConfig, decompose, raspen_solve, build_local_systems
from paper_2411_00546_b200.problems import EXTRA_CONFIGS, build_spec
cfg = EXTRA_CONFIGS["wide2x2"]
spec = build_spec(cfg, with_matrix=False)
dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
eng = build_local_systems(dec, spec)
for r in range(2):
    eng.set_profiling(True); eng.reset_stats()
    t0 = time.perf_counter()
    x, rep = raspen_solve(np.zeros(cfg.unknowns), dec, spec, ContinuationSchedule(1.0, 0.1, 1e-6), cfg=NewtonConfig(tol=1e-10), krylov_cfg=KrylovConfig(rel_tol=1e-8, max_iters=1000), inner_tol=1e-8)
    st = eng.stats()
    print(f"wide2x2 GPU: {time.perf_counter()-t0:.3f} s conv={rep.converged} outer={rep.outer_iters} gmres={rep.gmres_iters}", {k: round(v, 1) for k, v in st.items() if k.endswith('_ms')}, flush=True)
