"""Per-phase cycles of k_block_factor (build with OCP_PHASE_TIMING=1), config-4 factor."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
sys.argv = ["factor_bench.py", sys.argv[1] if len(sys.argv) > 1 else "cfg4", "1"]
exec(open("tools/factor_bench.py").read())
import os
lib = ctypes.CDLL(os.environ.get("OCP_LIB", "paper_2411_00546_b200/libocpgpu.so"))
buf = (ctypes.c_ulonglong * 16)()
lib.ocp_debug_phase(buf)
v = np.array(list(buf), dtype=float)[8:] / 2.0   # the counters cover the warm-up launch and the timed one
names = ["", "E2", "P2 row block", "P3a trailing", "P3b column block", "P1 pivot inverse",
         "store (TMA issue + wait read)", "E1 scale"]
tot = v[1:8].sum()
print(f"per launch, summed over the CTAs (cycles); with -DOCP_P1_SERIAL slot 0 is the pivot-step loop alone")
print(f"lookahead path (tile + pivot inverse, inside P3a): {v[0]:.3e} cycles")

for k in range(1, 8):
    print(f"{names[k]:28s} {100 * v[k] / tot:5.1f}%  {v[k]:.3e} cycles")
