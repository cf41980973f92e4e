"""Per-CTA phase timeline of the 2D p = 3 sweep kernel (an A/B build with -DADG_2P3_TIMING,
tools/build_ab.sh): thread 0 of every CTA stamps %clock64 at the phase boundaries and
%globaltimer at entry / exit; this prints the mean phase lengths of the last sweep of a
captured step graph and the spread of the CTA start / end times.

    python tools/cta_timeline.py --lib=tools/ab/lib_timing.so [steps]
"""

import ctypes
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1801_08682_b200 import _lib, scenarios  # noqa: E402
from paper_1801_08682_b200.parallel import SlabDriver  # noqa: E402

NAMES = ["entry", "loads issued", "tc words here", "corrector+Q", "lambda words", "picard", "fbar",
         "volume/qbar/smax", "records", "(barrier)", "threadfence", "atomic arrive"]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--lib=")]
    for a in sys.argv[1:]:
        if a.startswith("--lib="):
            _lib._lib = _lib.load_library(a[len("--lib="):])
    steps = int(args[0]) if args else 6
    cfg = bench.CONFIGS["cfg1"]
    d, L, p = cfg["d"], cfg["L"], cfg["p"]
    Q0 = scenarios.build(cfg["scenario"], d, L, p)
    drv = SlabDriver(Q0, d, L, p, 0, 1, 0)
    h = drv.handle
    drv.enqueue_step()
    drv.enqueue_step()
    torch.cuda.synchronize()
    out = (ctypes.c_double * 2)()
    for n in (4, 4, steps):
        h.call("adg_run_timed_ex", n, 0, out)
        print(f"{n} steps: {1e3 * out[0] / n:.2f} us/step")
    ptr, nbytes = h.buffer(99)
    t = torch.as_tensor(_lib.DeviceArray(ptr, (nbytes // 256, 32), "<f8", 0), device="cuda:0").cpu().numpy()
    clk = t[:, 1:13]
    dur = np.diff(clk, axis=1)
    print(f"CTAs {t.shape[0]}, mean Picard iterations {t[:, 13].mean():.2f}")
    for i, nm in enumerate(NAMES[1:]):
        print(f"  {NAMES[i]:>18s} -> {nm:<18s} mean {dur[:, i].mean():8.0f} clk   max {dur[:, i].max():8.0f}")
    its = t[:, 16:26]
    for i in range(9):
        m = (t[:, 13] > i)
        if m.sum():
            print(f"  iteration {i}: top -> next top   mean {(its[m, i + 1] - its[m, i]).mean():8.0f} clk over {m.sum()} CTAs")
    print(f"  iteration 2: top -> flux stored + votes {(t[:, 10] - its[:, 2]).mean():.0f}, barrier {(t[:, 11] - t[:, 10]).mean():.0f}, "
          f"vote words + derivative {(t[:, 12] - t[:, 11]).mean():.0f}, exchange + contraction + update {(t[:, 31] - t[:, 12]).mean():.0f}, "
          f"-> next top {(its[:, 3] - t[:, 31]).mean():.0f} clk")
    print(f"  first loop top after 'lambda words' stamp: {(its[:, 0] - t[:, 5]).mean():8.0f} clk; "
          f"last top -> 'picard' stamp {np.mean([t[i, 6] - its[i, int(t[i, 13])] for i in range(t.shape[0])]):8.0f} clk")
    b = t[:, 26:31]
    last = t[:, 14] == t.shape[0] - 1
    print(f"  grid barrier (multi-step kernel), non-last CTAs: records -> barrier entry {(b[~last, 0] - t[~last, 9]).mean():.0f}, "
          f"fence {(b[~last, 1] - b[~last, 0]).mean():.0f}, arrive atomic {(b[~last, 2] - b[~last, 1]).mean():.0f}, "
          f"spin {(b[~last, 3] - b[~last, 2]).mean():.0f} (min {(b[~last, 3] - b[~last, 2]).min():.0f}, max "
          f"{(b[~last, 3] - b[~last, 2]).max():.0f}), fence {(b[~last, 4] - b[~last, 3]).mean():.0f} clk")
    if last.any():
        print(f"  last CTA: fence {(b[last, 1] - b[last, 0]).mean():.0f}, arrive {(b[last, 2] - b[last, 1]).mean():.0f}, "
              f"time control {(b[last, 3] - b[last, 2]).mean():.0f}, fence + release {(b[last, 4] - b[last, 3]).mean():.0f} clk")
    ge = t[:, 15]
    print(f"  globaltimer: step entry spread {t[:, 0].max() - t[:, 0].min():.0f} ns; first entry -> last barrier exit "
          f"{ge.max() - t[:, 0].min():.0f} ns; barrier exit spread {ge.max() - ge.min():.0f} ns")
    print(f"  CTA lifetime (clock64)        mean {(clk[:, -1] - clk[:, 0]).mean():8.0f} clk   max "
          f"{(clk[:, -1] - clk[:, 0]).max():8.0f}")
    g0, g1 = t[:, 0], t[:, 15]
    print(f"  globaltimer: first entry -> last entry {g0.max() - g0.min():.0f} ns, first entry -> last exit "
          f"{g1.max() - g0.min():.0f} ns, mean lifetime {(g1 - g0).mean():.0f} ns")
    order = np.argsort(t[:, 14])
    print(f"  arrival order: first CTA exit at +{g1[order[0]] - g0.min():.0f} ns, last at +{g1[order[-1]] - g0.min():.0f} ns")
    drv.close()


if __name__ == "__main__":
    main()
