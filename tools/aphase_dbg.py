"""Per-phase cycles of the Arnoldi kernel, block 0 (build with OCP_PHASE_TIMING=1): config-4 solve."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
sys.argv = ["run_cfg.py", "cfg4", "1e-7", "1"]
exec(open("tools/run_cfg.py").read())
import os
lib = ctypes.CDLL(os.environ.get("OCP_LIB", "paper_2411_00546_b200/libocpgpu.so"))
buf = (ctypes.c_ulonglong * 24)()
lib.ocp_debug_phase(buf)
v = np.array(list(buf), dtype=float)[16:]
passes = 47206 + 5 * 2   # MGS passes of one config-4 solve (+ norm passes counted in phase 1..4)
names = ["sync+issue+TMA wait", "dot A,B + block reduce", "barrier wait", "grid sum", "publish + axpy + qv"]
for k in range(5):
    print(f"{names[k]:22s} {v[k]:.3e} cycles  ~{v[k] / passes / 1.965e3:.2f} us/pass")
