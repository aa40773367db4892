"""Per-phase cycles of k_block_factor (build with OCP_PHASE_TIMING=1), config-4 factor."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
sys.argv = ["factor_bench.py", sys.argv[1] if len(sys.argv) > 1 else "cfg4", "1"]
exec(open("tools/factor_bench.py").read())
lib = ctypes.CDLL("paper_2411_00546_b200/libocpgpu.so")
buf = (ctypes.c_ulonglong * 16)()
lib.ocp_debug_phase(buf)
v = np.array(list(buf), dtype=float)[8:]
names = ["", "E + first P1", "P2 row block", "P3a + lookahead P1", "P3b column block",
         "  warp 0: lookahead tile + P1", "  warp 0: tile loop", "  warp 4: tile loop"]
tot = v[1:5].sum()
print(f"trailing tile cycles (sum over all warps/tiles): {v[0]:.3e}  per tile: {v[0] / (256 * 79 * 28 * 5):.0f} (approx count)")
for k in range(1, 8):
    print(f"{names[k]:28s} {100 * v[k] / tot:5.1f}%  {v[k]:.3e} cycles")
