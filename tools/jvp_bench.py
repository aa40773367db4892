"""Time the stored-factor JVP solve alone at a config (after one RAS sweep):
average fused k_block_solve<2> launch time from the context's CUDA-event
stats.  OCP_LIB selects an experiment build of libocpgpu.so."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import ContinuationSchedule, NewtonConfig, build_local_systems, decompose  # noqa: E402
from paper_2411_00546_b200.problems import CONFIGS, build_spec  # noqa: E402
from paper_2411_00546_b200.schwarz import _jvp, _sweep  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = CONFIGS[name]
spec = build_spec(cfg, with_matrix=False)
dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
eng = build_local_systems(dec, spec)
x = eng.from_host(np.zeros(cfg.unknowns))
fac = eng.factor_store()
sched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min) if cfg.gamma < 1 else ContinuationSchedule.fixed(cfg.eps_min)
_sweep(eng, x, fac, sched, NewtonConfig(tol=1e-7))
d = eng.from_host(np.random.default_rng(1).standard_normal(cfg.unknowns))
for _ in range(5):
    out = _jvp(eng, fac, d)
eng.sync()
eng.set_profiling(True)
eng.reset_stats()
for _ in range(reps):
    out = _jvp(eng, fac, d)
eng.sync()
st = eng.stats()
print(f"{os.environ.get('OCP_LIB', 'default')}: jvp {st['jvp_ms'] / reps:.4f} ms, "
      f"solve {st['solve_ms'] / st['solve_launches']:.4f} ms, "
      f"{st['solve_bytes'] / st['solve_ms'] / 1e6:.0f} GB/s, norm {out.norm():.12e}")
