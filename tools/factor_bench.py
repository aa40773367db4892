"""Time the batched block factor alone: the RAS-preconditioner factorisation of all
subdomains of a config (one k_block_factor launch per call)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import build_local_systems, decompose  # noqa: E402
from paper_2411_00546_b200.linear_ras import RasPreconditioner  # noqa: E402
from paper_2411_00546_b200.problems import CONFIGS, build_spec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = CONFIGS[name]
spec = build_spec(cfg, with_matrix=False)
dec = decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap)
eng = build_local_systems(dec, spec)
x = eng.from_host(0.1 * np.random.default_rng(0).standard_normal(cfg.unknowns))
fac = eng.factor_store()
try:
    RasPreconditioner(eng, x, cfg.eps_min, fac)   # warm-up
except Exception:
    pass
eng.set_profiling(True)
eng.reset_stats()
for _ in range(reps):
    try:
        RasPreconditioner(eng, x, cfg.eps_min, fac)
    except Exception as exc:  # experiments may break the numerics
        print("note:", type(exc).__name__, str(exc)[:80])
st = eng.stats()
print(f"{name}: factor {st['factor_ms'] / st['factor_launches']:.3f} ms/launch, "
      f"{st['factor_flops'] / st['factor_ms'] / 1e9:.2f} TFLOP/s")
