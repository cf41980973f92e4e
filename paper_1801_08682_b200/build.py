"""Build the sm_100a CUDA libraries in-tree (nvcc cross-compiles without a GPU).

    python -m paper_1801_08682_b200.build [--force]

* ``libaderdg_b200.so``        the product library (include/aderdg_b200.h);
* ``libaderdg_b200_debug.so``  the same sources with ADG_DEBUG_CHECKS: face-record
  sweep stamps and slot bounds checked on every read, NaN-poisoned shared memory,
  jittered CTA barriers and reversed cell order (tests/test_gpu_debug.py).  The
  compute-sanitizer tools are closed on this GPU pool; these checks stand in for
  racecheck / initcheck / memcheck on the hot kernels.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libaderdg_b200.so")
OUT_DEBUG = os.path.join(HERE, "libaderdg_b200_debug.so")
SOURCES = [os.path.join(CSRC, "aderdg_capi.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".cuh")] + \
    [os.path.join(os.path.dirname(HERE), "include", "aderdg_b200.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-std=c++17", "-Xcompiler", "-fPIC", "-shared"]
VARIANTS = {OUT: [], OUT_DEBUG: ["-DADG_DEBUG_CHECKS"]}


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.exists(cand) or cand == "nvcc"):
            return cand
    return "nvcc"


def up_to_date(out):
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def build(force=False, verbose=False, debug=True):
    """Compile the product (and debug) library; the two nvcc runs go in parallel."""
    procs = []
    for out, extra in VARIANTS.items():
        if (out == OUT_DEBUG and not debug) or (not force and up_to_date(out)):
            continue
        cmd = [nvcc()] + NVCC_FLAGS + extra + ["-o", out] + SOURCES
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd)))
    for cmd, pr in procs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, cmd)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, debug="--no-debug" not in sys.argv)
