"""Short config-4 workload for ncu: one RAS sweep (continuation) + a few JVPs + MGS."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import ContinuationSchedule, NewtonConfig, build_local_systems, decompose  # noqa: E402
from paper_2411_00546_b200.problems import CONFIGS, build_spec  # noqa: E402
from paper_2411_00546_b200.schwarz import _jvp, _sweep  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
njvp = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS[name]
spec = build_spec(cfg, with_matrix=False)
dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
eng = build_local_systems(dec, spec)
x = eng.from_host(np.zeros(cfg.unknowns))
fac = eng.factor_store()
sched = ContinuationSchedule(cfg.eps0, cfg.gamma, cfg.eps_min) if cfg.gamma < 1 else ContinuationSchedule.fixed(cfg.eps_min)
fval, inner = _sweep(eng, x, fac, sched, NewtonConfig(tol=1e-7))
print("inner", max(inner), min(inner))
d = eng.from_host(np.random.default_rng(1).standard_normal(cfg.unknowns))
for _ in range(njvp):
    out = _jvp(eng, fac, d)
eng.sync()
print("norm", out.norm())
