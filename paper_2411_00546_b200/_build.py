"""Compile the CUDA sources into the in-tree ``libocpgpu.so`` (sm_100a).

Called by ``__graft_entry__.build()`` and by ``python -m
paper_2411_00546_b200._build``.  The library is built in-tree so the ``.so``
travels to the GPU box with the repo snapshot.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libocpgpu.so")
SOURCES = ["ocp_abi.cu", "ocp_kernels.cu", "ocp_krylov.cu", "ocp_global.cu", "ocp_block.cu",
           "ocp_block_narrow.cu"]
NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-shared",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def sources():
    return [os.path.join(CSRC, s) for s in SOURCES]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "ocp_gpu.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force=False, verbose=False):
    if not force and not stale():
        return LIB
    extra = ["-DOCP_PHASE_TIMING"] if os.environ.get("OCP_PHASE_TIMING") else []
    extra += os.environ.get("OCP_EXTRA_NVCC", "").split()   # experiments only
    cmd = [nvcc()] + NVCC_FLAGS + extra + ["-o", LIB] + sources()
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=CSRC)
    return LIB


TOOLS = {"fp64_peak": "fp64_peak.cu", "dmma_peak": "dmma_peak.cu", "rn_check": "rn_check.cu"}


def build_tools(verbose=False):
    """Peak probes used by bench.py for the FP64 roofline denominator, and the
    bitwise check of the branch-free division / square root (tests, -m gpu)."""
    tdir = os.path.join(os.path.dirname(HERE), "tools")
    for exe, src in TOOLS.items():
        cmd = [nvcc(), "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-I", CSRC,
               "-o", os.path.join(tdir, exe), os.path.join(tdir, src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    build_tools(verbose=True)
