"""Build the sm_100a CUDA library in-tree (nvcc cross-compiles without a GPU).

    python -m paper_1801_08682_b200.build
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libaderdg_b200.so")
SOURCES = [os.path.join(CSRC, "aderdg_capi.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "aderdg_kernels.cuh"), os.path.join(CSRC, "aderdg_sweep_v2.cuh"),
                  os.path.join(CSRC, "aderdg_sweep_ho.cuh"),
                  os.path.join(CSRC, "aderdg_limiter.cuh"),
                  os.path.join(os.path.dirname(HERE), "include", "aderdg_b200.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-std=c++17", "-Xcompiler", "-fPIC", "-shared"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.exists(cand) or cand == "nvcc"):
            return cand
    return "nvcc"


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    cmd = [nvcc()] + NVCC_FLAGS + ["-o", OUT] + SOURCES
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
