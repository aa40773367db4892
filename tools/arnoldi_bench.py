"""Time one Arnoldi step (ocp_arnoldi: MGS against j+1 basis vectors) at config-4 size."""
import ctypes
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2411_00546_b200 import build_local_systems, decompose  # noqa: E402
from paper_2411_00546_b200.problems import CONFIGS, build_spec  # noqa: E402

cfg = CONFIGS["cfg4"]
spec = build_spec(cfg, with_matrix=False)
eng = build_local_systems(decompose(spec.grid, cfg.s1, cfg.s2, cfg.overlap), spec)
n = cfg.unknowns
j = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(0)
Q = eng.buffer(8 * n * (j + 2))
for c in range(j + 1):
    v = rng.standard_normal(n)
    eng.check(eng.lib.ocp_h2d(eng.ctx, ctypes.c_void_p(Q.addr + 8 * n * c), v.ctypes.data_as(ctypes.c_void_p), 8 * n), "h2d")
w = eng.from_host(rng.standard_normal(n))
h = np.zeros(j + 2)
hp = h.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
for rep in range(2):
    eng.sync()
    t0 = time.perf_counter()
    for _ in range(10):
        eng.check(eng.lib.ocp_arnoldi(eng.ctx, n, ctypes.c_void_p(Q.addr), n, j, w.ptr, hp), "arnoldi")
    dt = (time.perf_counter() - t0) / 10
print(f"j={j}: {dt * 1e3:.3f} ms per Arnoldi step, {dt / (j + 2) * 1e6:.2f} us per MGS pass "
      f"(HBM floor {n * 8 / 6.5456e12 * 1e6:.2f} us)")
