"""Golden vectors of the reference's subcell-limited straightforward driver.

Runs only in the build container (imports ``/root/reference/pkg/src/aderdg``):

    python tests/golden/make_limiter_golden.py [case ...]

Each case builds the reference grid (periodic, ``storage="spacetime"``), fills
``cell.Q`` from a seeded scenario of ``paper_1801_08682_b200/scenarios.py``,
attaches ``SubcellLimiter(system, basis, grid, cfl=0.9)``
(``src/limiter.py:87-108``) and runs ``Driver(..., "straightforward",
limiter=lim)`` (``src/scheduler.py:230-313``), optionally with a Peano
traversal (``src/mesh.py:246-286``).  Stored in ``tests/golden/lim_<case>.npz``:
per-step records (step, T, dt_old, dt_new, dt_adm, troubled), the final state,
the final troubled flags, and the error (class, message, cell) if one was
raised.
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from paper_1801_08682_b200 import scenarios  # noqa: E402

# name: (scenario, scenario kwargs, d, L, p, steps, driver kwargs, tc kwargs)
CASES = {
    "tube_d2_L2_p2": ("shocktube", {}, 2, 2, 2, 12, {}, {}),
    "tube_d2_L2_p3": ("shocktube", {"noise": 1e-2, "seed": 4}, 2, 2, 3, 15, {}, {}),
    "tube_d2_L2_p3_peano": ("shocktube", {"noise": 1e-2, "seed": 4}, 2, 2, 3, 10,
                            {"traversal": "peano"}, {}),
    "tube_d2_L2_p5_forced": ("shocktube", {}, 2, 2, 5, 8, {}, {"forced_dt": 1e-3}),
    "tube_d3_L1_p3": ("shocktube", {}, 3, 1, 3, 6, {}, {}),
    "tube_d3_L1_p2_creeping": ("shocktube", {"pressure_ratio": 30.0}, 3, 1, 2, 6, {},
                               {"averaging": "creeping"}),
    "bump_d3_L1_p7_noisy": ("bump", {"noise": 5e-2, "seed": 2}, 3, 1, 7, 4, {}, {}),
    "tube_d2_L1_p9": ("shocktube", {}, 2, 1, 9, 5, {}, {}),
    # outflow Sod, the reference's own limiter tests (tests/test_limiter.py:130-151,
    # tests/test_acceptance.py:202-229)
    "sod_d2_L2_p2": ("sod", {}, 2, 2, 2, 30, {}, {}),
    "sod_d2_L2_p3": ("sod", {}, 2, 2, 3, 30, {}, {}),
    "sod_d2_L2_p3_100": ("sod", {}, 2, 2, 3, 100, {}, {}),
    "sod_d3_L1_p2": ("sod", {}, 3, 1, 2, 10, {}, {}),
    "sod_d2_L2_p4_peano": ("sod", {}, 2, 2, 4, 12, {"traversal": "peano"}, {}),
}


def run_case(name, spec):
    from aderdg import (Driver, EulerSystem, Kernels, NumericalError, PredictorFailureError,
                        TimeControl, build_grid, make_basis)
    from aderdg.limiter import SubcellLimiter
    scen, skw, d, L, p, steps, dkw, tkw = spec
    Q0 = scenarios.build(scen, d, L, p, **skw)
    system = EulerSystem(d)
    basis = make_basis(p)
    boundary = "outflow" if scen in scenarios.OUTFLOW else "periodic"
    grid = build_grid(d, L, p, system.m, boundary=boundary, storage="spacetime", budget_bytes=1 << 40)
    for c in grid.cells:
        c.Q[...] = Q0[c.index]
    lim = SubcellLimiter(system, basis, grid, cfl=0.9)
    kernels = Kernels(system, basis, grid, None, cfl=0.9)
    error = None
    driver = None
    t0 = time.time()
    try:
        driver = Driver(grid, kernels, TimeControl(c_dt=0.99, **tkw), "straightforward",
                        limiter=lim, **dkw)
        for _ in range(steps):
            driver.step()
    except (NumericalError, PredictorFailureError) as e:
        error = {"class": type(e).__name__, "message": str(e),
                 "cell": getattr(e, "cell_index", None)}
    wall = time.time() - t0
    recs = driver.step_records if driver is not None else []
    rec_arr = np.array([[r["step"], r["T"], r["dt_old"], r["dt_new"], r["dt_adm"], r["troubled"]]
                        for r in recs], dtype=np.float64).reshape(-1, 6)
    out = {
        "records": rec_arr,
        "Q0_sum": np.array([np.sum(Q0), np.sum(np.abs(Q0))]),
        "Q_final": np.stack([c.Q for c in grid.cells]),
        "troubled_final": np.array([bool(c.troubled) for c in grid.cells]),
        "meta": np.array(json.dumps({"scenario": scen, "scenario_kwargs": skw, "boundary": boundary,
                                     "d": d, "L": L,
                                     "p": p, "steps": steps, "driver_kwargs": dkw,
                                     "tc_kwargs": tkw, "error": error, "wall_s": wall})),
    }
    if "traversal" in dkw:
        out["order"] = np.asarray(driver.order if driver is not None else [], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, f"lim_{name}.npz"), **out)
    print(f"lim_{name}: {wall:.1f}s steps={len(recs)} troubled={rec_arr[:, 5].astype(int).tolist()} "
          f"error={error}", flush=True)


def main():
    names = sys.argv[1:] or list(CASES)
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    for n in names:
        run_case(n, CASES[n])


if __name__ == "__main__":
    main()
