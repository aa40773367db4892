"""Per-subdomain durations of one k_block_factor launch (build with
OCP_PHASE_TIMING; OCP_LIB selects it): which subdomain shapes bound the
launch, and how busy the SMs are over it."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.argv = ["factor_bench.py", sys.argv[1] if len(sys.argv) > 1 else "cfg4", "1"]
exec(open("tools/factor_bench.py").read())
lib = ctypes.CDLL(os.environ.get("OCP_LIB", "paper_2411_00546_b200/libocpgpu.so"))
I = eng.num_subdomains
buf = (ctypes.c_longlong * (3 * I))()
lib.ocp_debug_subt(buf, I)
t = np.array(list(buf), dtype=np.int64).reshape(I, 3)
dur = t[:, 1] - t[:, 0]
shape = [(int(r[1]), int(r[2])) for r in eng.rects] if hasattr(eng, "rects") else None
print(f"subdomains {I}: duration kcycles min {dur.min()/1e3:.0f} median {np.median(dur)/1e3:.0f} max {dur.max()/1e3:.0f}")
order = np.argsort(-dur)[:8]
for i in order:
    print(f"  sub {i:4d} rect {eng.rects[i][:6].tolist()} {dur[i]/1e3:.0f} kcycles on SM {t[i, 2]}")
per_sm = {}
for i in range(I):
    per_sm.setdefault(int(t[i, 2]), []).append(dur[i])
loads = np.array([sum(v) for v in per_sm.values()])
print(f"SM load kcycles: max {loads.max()/1e3:.0f} mean {loads.mean()/1e3:.0f} (balance {loads.mean()/loads.max():.2f})")
