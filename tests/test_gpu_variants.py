"""GPU parity of the selectable kernel variants (ADG_KERNEL=<n>, read by adg_create).

The defaults are covered by test_gpu_parity.py; every A/B variant that stays in the
library (the measured alternatives DESIGN.md §3 reports) must meet the same bar:
relative L-inf <= 1e-10 against the CPU oracle on seeded noisy states, identical
rerun steps.
"""

import os

import pytest

import aderdg_oracle as O
from conftest import make_system, rel_linf
from paper_1801_08682_b200 import Driver, Kernels, TimeControl, build_grid, make_basis, scenarios

pytestmark = pytest.mark.gpu
TOL = 1e-10

# (variant, d, L, p, steps, seed): p=3 slice loops, p=5 layouts, high-order engines / TMEM
CASES = [
    (21, 3, 2, 3, 3, 7),   # p=3: slice at a time (A1S)
    (22, 3, 2, 3, 3, 7),   # p=3: pipelined, DMMAs after the barrier
    (14, 3, 2, 3, 3, 7),   # p=3: axis 1 through shared memory
    (30, 3, 1, 5, 3, 1),   # p=5: pencil Picard loop
    (32, 3, 1, 5, 3, 1),   # p=5: C-order node mapping
    (2, 3, 1, 5, 3, 1),    # p=5: time split
    (40, 3, 1, 7, 3, 4),   # p=7: TMEM old iterate (default)
    (41, 3, 1, 7, 3, 4),   # p=7: local-memory time line
    (42, 3, 1, 7, 3, 4),   # p=7: TMEM divergence history
    (18, 3, 1, 7, 3, 4),   # p=7: constant-bank line engine
    (40, 3, 1, 9, 2, 8),   # p=9: TMEM old iterate
    (42, 3, 1, 9, 2, 8),   # p=9: TMEM divergence history
    (15, 3, 1, 9, 2, 8),   # p=9: DMMA tile engine
    (45, 3, 1, 9, 2, 8),   # p=9: half a cell per SM on a 2-CTA cluster (distributed shared memory)
    (45, 3, 1, 7, 3, 4),   # p=7: the same
    (1, 3, 1, 5, 3, 1),    # first-generation kernel
]


@pytest.mark.parametrize("var,d,L,p,steps,seed", CASES)
def test_variant_matches_oracle(cuda_ok, var, d, L, p, steps, seed):
    Q0 = scenarios.build("bump", d, L, p, seed=seed, noise=1e-2)
    old = os.environ.get("ADG_KERNEL")
    os.environ["ADG_KERNEL"] = str(var)
    try:
        system = make_system(d, None)
        grid = build_grid(d, L, p, system.m)
        grid.Q[...] = Q0
        drv = Driver(grid, Kernels(system, make_basis(p), grid, None, cfl=0.9), TimeControl(c_dt=0.99),
                     "fused", host_sync="run")
    finally:
        if old is None:
            os.environ.pop("ADG_KERNEL", None)
        else:
            os.environ["ADG_KERNEL"] = old
    drv.run(steps=steps)
    ora = O.FusedDriver(Q0.copy(), d, p, L)
    ora.run(steps)
    assert rel_linf(drv.grid.Q, ora.Q) <= TOL, f"variant {var}"
    assert [r["reruns"] for r in drv.step_records] == [r["reruns"] for r in ora.step_records]
