"""Per-CTA timeline of sweep_kernel_p5 (A/B build with -DADG_P5_TIMING, tools/build_ab.sh): cost of
the per-cell TMEM allocation / release and the occupancy of the SM's two CTA slots over a sweep
(would a persistent CTA per slot, looping over cells, pay?).

    python tools/p5_timeline.py --lib=tools/ab/lib_p5timing.so [config=cfg3_p5]
"""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1801_08682_b200 import _lib, scenarios  # noqa: E402
from paper_1801_08682_b200.parallel import SlabDriver  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--lib=")]
    for a in sys.argv[1:]:
        if a.startswith("--lib="):
            _lib._lib = _lib.load_library(a[len("--lib="):])
    cfg = bench.CONFIGS[args[0] if args else "cfg3_p5"]
    d, L, p = cfg["d"], cfg["L"], cfg["p"]
    Q0 = scenarios.build(cfg["scenario"], d, L, p)
    drv = SlabDriver(Q0, d, L, p, 0, 1, 0)
    h = drv.handle
    for _ in range(3):
        drv.enqueue_step()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    h.call("adg_phase_sweep")
    ev[1].record()
    h.call("adg_phase_finish")
    torch.cuda.synchronize()
    ptr, nbytes = h.buffer(98)
    t = torch.as_tensor(_lib.DeviceArray(ptr, (nbytes // 64, 8), "<f8", 0), device="cuda:0").cpu().numpy()
    life = t[:, 7] - t[:, 0]
    print(f"sweep {1e3 * ev[0].elapsed_time(ev[1]):.1f} us, {t.shape[0]} CTAs, mean CTA lifetime {life.mean() / 1e3:.2f} us "
          f"(globaltimer), entry -> TMEM alloc {(t[:, 2] - t[:, 1]).mean():.0f} clk")
    print(f"tcgen05.alloc (+ relinquish) {(t[:, 3] - t[:, 2]).mean():.0f} clk (max {(t[:, 3] - t[:, 2]).max():.0f}), "
          f"tcgen05.dealloc {(t[:, 5] - t[:, 4]).mean():.0f} clk (max {(t[:, 5] - t[:, 4]).max():.0f})")
    clk_ns = 1.965
    pic = (t[:, 4] - t[:, 3]) / clk_ns
    pro = (t[:, 2] - t[:, 1]) / clk_ns
    print(f"phases (ns): prologue up to the allocation {pro.mean():.0f}, Picard loop + final flux {pic.mean():.0f} "
          f"(min {pic.min():.0f}, max {pic.max():.0f}), tail {(life - pro - pic).mean() - (t[:, 5] - t[:, 4]).mean() / clk_ns:.0f}")
    wall = t[:, 7].max() - t[:, 0].min()
    sms = np.unique(t[:, 6])
    busy = np.array([life[t[:, 6] == s].sum() for s in sms])
    print(f"first entry -> last exit {wall / 1e3:.1f} us on {len(sms)} SMs; CTA-slot occupancy (sum of lifetimes / 2 slots x wall): "
          f"mean {np.mean(busy / (2 * wall)):.4f}, min {np.min(busy / (2 * wall)):.4f}")
    gaps = []
    for s in sms[:16]:
        m = t[:, 6] == s
        e0, e1 = np.sort(t[m, 0]), np.sort(t[m, 7])
        # a slot is refilled at the entry that follows an exit: k-th exit -> (k+2)-th entry
        gaps.append(np.mean(e0[2:] - e1[:-2]))
    print(f"exit of a CTA -> entry of the CTA that takes its slot: {np.mean(gaps):.0f} ns (16 SMs)")
    drv.close()


if __name__ == "__main__":
    main()
