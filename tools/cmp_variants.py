"""A/B numerics: run the same seeded BASELINE-type state through two ADG_KERNEL
variants step by step and print the largest relative difference of Q per step.
    python tools/cmp_variants.py A B [d L p steps]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_08682_b200 import Driver, EulerSystem, Kernels, TimeControl, build_grid, make_basis, scenarios


def make(var, Q0, d, L, p):
    os.environ["ADG_KERNEL"] = str(var)
    grid = build_grid(d, L, p, d + 2)
    grid.Q[...] = Q0
    return grid, Driver(grid, Kernels(EulerSystem(d), make_basis(p), grid, None), TimeControl(), "fused",
                        device=0, host_sync="step")


def main():
    a, b = sys.argv[1], sys.argv[2]
    d, L, p, steps = (int(x) for x in (sys.argv[3:7] if len(sys.argv) > 6 else (3, 1, 5, 4)))
    Q0 = scenarios.build("bump", d, L, p)
    ga, da = make(a, Q0, d, L, p)
    gb, db = make(b, Q0, d, L, p)
    for s in range(steps):
        da.step(); db.step()
        qa, qb = np.array(ga.Q), np.array(gb.Q)
        err = np.abs(qa - qb)
        i = np.unravel_index(np.argmax(err), err.shape)
        print(f"step {s + 1}: rel {err.max() / np.abs(qa).max():.3e} at {i}; picard {da.step_records[-1]} | {db.step_records[-1]}",
              flush=True)


if __name__ == "__main__":
    main()
