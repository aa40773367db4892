"""Build an experiment variant of libocpgpu.so into tools/exp_<name>/ with extra
nvcc flags (e.g. -DOCP_BS_PF_LINES=4); select it at run time with OCP_LIB."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2411_00546_b200 import _build  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"exp_{name}")
os.makedirs(out, exist_ok=True)
cmd = [_build.nvcc()] + _build.NVCC_FLAGS + flags + ["-o", os.path.join(out, "libocpgpu.so")] + _build.sources()
subprocess.run(cmd, check=True, cwd=_build.CSRC)
print(os.path.join(out, "libocpgpu.so"))
