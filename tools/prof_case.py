"""A bench configuration's steps as plain stream launches, for ncu (tools/profile_r02.sh).

    python tools/prof_case.py <config> [warm_steps] [profiled_steps]

Runs ``warm_steps`` untimed steps (the first carries the priming sweep), then
``profiled_steps`` more; every step launches the rerun pass (early exit without a
rerun), the sweep and the time-control kernel on the handle's stream (no CUDA graph,
so ncu sees each launch).  Launch order: priming sweep, finish, then per step
rerun-pass sweep, sweep, finish: skip 1 + 2 * warm_steps sweep launches to reach the
profiled steps.
"""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402
from paper_1801_08682_b200 import scenarios  # noqa: E402
from paper_1801_08682_b200.parallel import SlabDriver  # noqa: E402


def main():
    name = sys.argv[1]
    warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    prof = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    cfg = bench.CONFIGS[name]
    d, L, p = cfg["d"], cfg["L"], cfg["p"]
    Q0 = scenarios.build(cfg["scenario"], d, L, p)
    drv = SlabDriver(Q0, d, L, p, 0, 1, 0)
    for _ in range(warm + prof):
        drv.enqueue_step()
    drv.handle.call("adg_sync")
    print(f"{name}: {warm} + {prof} steps, step count {drv.handle.lib.adg_step_count(drv.handle.h)}")
    drv.close()


if __name__ == "__main__":
    main()
