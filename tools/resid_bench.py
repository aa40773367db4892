"""Time the full-set local-residual stencil (k_residual) at a config: average
launch time and algorithmic GB/s (48 B per local point) over several RAS
sweeps, from the context's CUDA-event stats.  OCP_LIB selects an experiment
build of libocpgpu.so."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import ContinuationSchedule, NewtonConfig, build_local_systems, decompose  # noqa: E402
from paper_2411_00546_b200.problems import CONFIGS, build_spec  # noqa: E402
from paper_2411_00546_b200.schwarz import _sweep  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = CONFIGS[name]
spec = build_spec(cfg, with_matrix=False)
dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
eng = build_local_systems(dec, spec)
x = eng.from_host(np.zeros(cfg.unknowns))
fac = eng.factor_store()
sched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min) if cfg.gamma < 1 else ContinuationSchedule.fixed(cfg.eps_min)
fval, _ = _sweep(eng, x, fac, sched, NewtonConfig(tol=1e-7))
eng.sync()
eng.set_profiling(True)
eng.reset_stats()
for _ in range(reps):
    fval, inner = _sweep(eng, x, fac, sched, NewtonConfig(tol=1e-7))
eng.sync()
st = eng.stats()
ms = st["resid_ms"] / max(st["resid_launches"], 1)
print(f"{os.environ.get('OCP_LIB', 'default')}: resid {ms * 1e3:.1f} us x {st['resid_launches']:.0f}, "
      f"{st['resid_bytes'] / st['resid_ms'] / 1e6:.0f} GB/s, inner {max(inner)}, "
      f"fval norm {fval.norm():.17e}")
