"""Per-launch CUDA-event times of a bench configuration's sweeps (stream launches and
the captured step graph), to cross-check bench.py against ncu's launch list.

    python tools/time_case.py <config> [steps]
"""

import ctypes
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1801_08682_b200 import _lib, scenarios  # noqa: E402
from paper_1801_08682_b200.parallel import SlabDriver  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--lib=")]
    for a in sys.argv[1:]:
        if a.startswith("--lib="):          # an A/B build (tools/build_ab.sh) instead of the product
            _lib._lib = _lib.load_library(a[len("--lib="):])
            print(f"library {a[len('--lib='):]}")
    name = args[0]
    steps = int(args[1]) if len(args) > 1 else 4
    cfg = bench.CONFIGS[name]
    d, L, p = cfg["d"], cfg["L"], cfg["p"]
    Q0 = scenarios.build(cfg["scenario"], d, L, p)
    drv = SlabDriver(Q0, d, L, p, 0, 1, 0)
    h = drv.handle
    drv.enqueue_step()
    drv.enqueue_step()
    torch.cuda.synchronize()
    # stream launches, events around each sweep launch
    for _ in range(steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        h.call("adg_phase_rerun")
        ev[1].record()
        h.call("adg_phase_sweep")
        ev[2].record()
        h.call("adg_phase_finish")
        ev[3].record()
        torch.cuda.synchronize()
        print(f"stream: rerun {ev[0].elapsed_time(ev[1]):.3f} sweep {ev[1].elapsed_time(ev[2]):.3f} "
              f"finish {ev[2].elapsed_time(ev[3]):.3f} ms", flush=True)
    for flags in (0, _lib.ADG_TIMED_KERNEL_EVENTS):
        out = (ctypes.c_double * 2)()
        t0 = time.perf_counter()
        h.call("adg_run_timed_ex", 2, flags, out)
        print(f"graph flags={flags}: segment {out[0] / 2:.3f} ms/step, kernels {out[1] / 2:.3f} ms/step, "
              f"wall {(time.perf_counter() - t0) * 500:.3f} ms/step", flush=True)
    drv.close()


if __name__ == "__main__":
    main()
