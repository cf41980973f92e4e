"""GPU parity of the subcell FV limiter (csrc/aderdg_limiter.cuh) through the C ABI.

* against the reference itself: ``tests/golden/lim_*.npz`` were written by
  ``Driver(..., "straightforward", limiter=SubcellLimiter(...))`` of the
  reference (``tests/golden/make_limiter_golden.py``); the GPU run must match
  the final state to 1e-10 relative L-inf (north-star tolerance), the dt log
  to 1e-10, and the per-step troubled counts and final troubled flags exactly;
* against the oracle (oracle/limiter_oracle.py) on other seeds, sizes and the
  advection plug-in;
* the reference's mode restriction (tests/test_limiter.py:170-176).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_linf

pytestmark = pytest.mark.gpu

CASES = sorted(f[4:-4] for f in os.listdir(GOLDEN) if f.startswith("lim_") and f.endswith(".npz"))
TOL = 1e-10


def gpu_run(Q0, d, L, p, steps, velocity=None, traversal="lexicographic", tc_kwargs=None,
            boundary="periodic"):
    from paper_1801_08682_b200 import (AdvectionSystem, Driver, EulerSystem, Kernels, SubcellLimiter,
                                       TimeControl, build_grid, make_basis)
    system = EulerSystem(d) if velocity is None else AdvectionSystem(d, velocity)
    grid = build_grid(d, L, p, system.m, boundary=boundary)
    grid.Q[...] = Q0
    basis = make_basis(p)
    lim = SubcellLimiter(system, basis, grid, cfl=0.9)
    drv = Driver(grid, Kernels(system, basis, grid, None), TimeControl(**(tc_kwargs or {})),
                 "straightforward", traversal=traversal, limiter=lim, device=0, host_sync="run")
    drv.run(steps=steps)
    return drv, grid


@pytest.mark.parametrize("name", CASES)
def test_limiter_matches_reference(cuda_ok, name):
    from paper_1801_08682_b200 import scenarios
    g = np.load(os.path.join(GOLDEN, f"lim_{name}.npz"))
    meta = json.loads(str(g["meta"]))
    d, L, p = meta["d"], meta["L"], meta["p"]
    Q0 = scenarios.build(meta["scenario"], d, L, p, **meta["scenario_kwargs"])
    trav = g["order"] if "order" in g else meta["driver_kwargs"].get("traversal", "lexicographic")
    drv, grid = gpu_run(Q0, d, L, p, meta["steps"], traversal=trav, tc_kwargs=meta["tc_kwargs"],
                        boundary=meta.get("boundary", "periodic"))
    assert rel_linf(grid.Q, g["Q_final"]) <= TOL
    rec = np.array([[r["step"], r["T"], r["dt_old"], r["dt_new"], r["dt_adm"], r["troubled"]]
                    for r in drv.step_records])
    assert np.array_equal(rec[:, 5], g["records"][:, 5])
    assert np.allclose(rec[:, 1:5], g["records"][:, 1:5], rtol=TOL, atol=0)
    assert dict(drv.troubled_by_step) == {int(s): int(t) for s, t in g["records"][:, [0, 5]] if t}
    assert np.array_equal(drv.troubled_flags(), g["troubled_final"])
    drv.close()


@pytest.mark.parametrize("scen,kw,d,L,p,steps,vel", [
    ("shocktube", {"noise": 2e-2, "seed": 9}, 2, 2, 4, 10, None),
    ("shocktube", {"noise": 1e-2, "seed": 3}, 3, 2, 3, 3, None),
    ("shocktube", {"pressure_ratio": 50.0}, 2, 2, 1, 12, None),
    ("shocktube", {}, 2, 2, 0, 10, None),
    ("gauss", {"noise": 0.3, "seed": 2}, 2, 2, 3, 6, (1.0, 0.5)),
    ("sod", {}, 3, 2, 2, 4, None),
])
def test_limiter_matches_oracle(cuda_ok, scen, kw, d, L, p, steps, vel):
    import aderdg_oracle as O  # noqa: F401  (sys.path set by conftest)
    import limiter_oracle as LO
    from paper_1801_08682_b200 import scenarios
    Q0 = scenarios.build(scen, d, L, p, **kw)
    bnd = "outflow" if scen in scenarios.OUTFLOW else "periodic"
    ora = LO.LimitedStraightforwardDriver(Q0.copy(), d, p, L, velocity=vel, boundary=bnd)
    with np.errstate(all="ignore"):
        ora.run(steps)
    drv, grid = gpu_run(Q0, d, L, p, steps, velocity=vel, boundary=bnd)
    assert rel_linf(grid.Q, ora.Q) <= TOL
    assert [r["troubled"] for r in drv.step_records] == [r["troubled"] for r in ora.step_records]
    assert np.array_equal(drv.troubled_flags(), ora.troubled)
    drv.close()


@pytest.mark.parametrize("p,steps", [(2, 30), (3, 30), (3, 100)])
def test_limited_sod_stays_admissible(cuda_ok, p, steps):
    """reference tests/test_limiter.py:130-151 and test_acceptance.py:202-229:
    outflow Sod with the limiter; limiting happens and every final state is
    admissible."""
    from paper_1801_08682_b200 import EulerSystem, scenarios
    Q0 = scenarios.build("sod", 2, 2, p)
    drv, grid = gpu_run(Q0, 2, 2, p, steps, boundary="outflow")
    assert sum(drv.troubled_by_step.values()) >= 1
    assert EulerSystem(2).is_admissible(grid.Q)
    drv.close()
