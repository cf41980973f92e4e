"""Generate golden vectors by running the REFERENCE implementation itself.

Runs only in the build container, where ``/root/reference`` exists:

    python tests/golden/make_golden.py [case ...]     # default: all small cases
    python tests/golden/make_golden.py --big          # BASELINE-size runs (minutes each)

For every case it builds the reference grid (``build_grid`` with an explicit
budget, ``src/mesh.py:167-243``), fills ``cell.Q`` from the seeded scenario in
``paper_1801_08682_b200/scenarios.py``, runs ``Driver(..., "fused")`` (or the
straightforward three-sweep driver for the ``sf_*`` cases, ``storage="spacetime"``)
(``src/scheduler.py:92-313``) and stores under ``tests/golden/<case>.npz``:

* ``records``: per step (step, T, dt_old, dt_new, dt_adm, reruns);
* ``Q_final`` (small cases) or ``Q_sample`` + ``sample_cells`` (large cases:
  every 97th cell) plus per-component sums/max of the final state;
* ``Q0_sum``: checksum of the initial state (guards scenario drift);
* ``picard``: Picard-iteration histogram observed in ``Kernels.predict``
  (``src/kernels.py:86-97``), counted by wrapping ``system.flux``;
* ``error``: if the reference raised, its class, message, cell and step.

The scenario builders are the harness's (the reference has no random states,
``src/cli.py:4-5``); the same array is later fed to the GPU path.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REPO)
sys.path.insert(0, REF_SRC)

from paper_1801_08682_b200 import scenarios  # noqa: E402

# name: (scenario, d, L, p, steps, extra driver kwargs, tc kwargs, store full Q)
SMALL = {
    "bump_d2_L2_p3": ("bump", 2, 2, 3, 10, {}, {}, True),
    "bump_d2_L3_p3_cfg1": ("bump", 2, 3, 3, 20, {}, {}, True),
    "bump_d2_L1_p0": ("bump", 2, 1, 0, 6, {}, {}, True),
    "bump_d2_L2_p1": ("bump", 2, 2, 1, 8, {}, {}, True),
    "bump_d2_L1_p9": ("bump", 2, 1, 9, 4, {}, {}, True),
    "bump_d2_L2_p6": ("bump", 2, 2, 6, 4, {}, {}, True),
    "bump_d3_L1_p3": ("bump", 3, 1, 3, 5, {}, {}, True),
    "bump_d3_L1_p2": ("bump", 3, 1, 2, 5, {}, {}, True),
    "bump_d3_L1_p5": ("bump", 3, 1, 5, 4, {}, {}, True),
    "bump_d3_L2_p3": ("bump", 3, 2, 3, 4, {}, {}, False),
    "fourier_d3_L1_p4": ("fourier", 3, 1, 4, 3, {}, {}, True),
    "wave_d2_L1_p2_spike": ("wave", 2, 1, 2, 10, {"spike_step": 4}, {}, True),
    "wave_d2_L1_p3_inject": ("wave", 2, 1, 3, 4, {"inject_rerun": True}, {}, True),
    "wave_d2_L2_p3_forced": ("wave", 2, 2, 3, 10, {}, {"forced_dt": 2e-4}, True),
    "wave_d3_L1_p2_creeping": ("wave", 3, 1, 2, 5, {}, {"averaging": "creeping"}, True),
    "uniform_d2_L1_p2": ("uniform", 2, 1, 2, 5, {}, {}, True),
    # straightforward (three-sweep) driver, src/scheduler.py:230-313
    "sf_bump_d2_L2_p3": ("bump", 2, 2, 3, 8, {"mode": "straightforward"}, {}, True),
    "sf_bump_d3_L1_p3": ("bump", 3, 1, 3, 5, {"mode": "straightforward"}, {}, True),
    "sf_wave_d2_L2_p3_forced": ("wave", 2, 2, 3, 10, {"mode": "straightforward"}, {"forced_dt": 2e-4}, True),
    "sf_bump_d3_L1_p5_creeping": ("bump", 3, 1, 5, 4, {"mode": "straightforward"}, {"averaging": "creeping"}, True),
    "sf_wave_d2_L1_p2_spike": ("wave", 2, 1, 2, 8, {"mode": "straightforward", "spike_step": 4}, {}, True),
    # AdvectionSystem(d, (1.0, 0.5, 0.25)[:d]) on the gaussian-advect profile (src/cli.py:139-142)
    "adv_gauss_d2_L2_p3": ("gauss", 2, 2, 3, 10, {}, {}, True),
    "adv_gauss_d2_L1_p0": ("gauss", 2, 1, 0, 6, {}, {}, True),
    "adv_gauss_d2_L2_p2_forced": ("gauss", 2, 2, 2, 10, {}, {"forced_dt": 1e-3}, True),
    "adv_gauss_d2_L1_p3_inject": ("gauss", 2, 1, 3, 4, {"inject_rerun": True}, {}, True),
    "adv_gauss_d3_L1_p5": ("gauss", 3, 1, 5, 4, {}, {}, True),
    "adv_gauss_d3_L1_p9": ("gauss", 3, 1, 9, 3, {}, {}, True),
    "adv_noise_d3_L2_p3": ("gauss_noise", 3, 2, 3, 5, {}, {}, True),
    "sf_adv_gauss_d2_L2_p3": ("gauss", 2, 2, 3, 8, {"mode": "straightforward"}, {}, True),
    "sf_adv_gauss_d3_L1_p4_creeping": ("gauss", 3, 1, 4, 4, {"mode": "straightforward"}, {"averaging": "creeping"}, True),
    # outflow boundaries (src/mesh.py:216-231, kernels.py:124-127), Sod without limiter
    "sod_d2_L2_p0": ("sod", 2, 2, 0, 12, {}, {}, True),
    "sod_d2_L2_p1": ("sod", 2, 2, 1, 6, {}, {}, True),
    "sod_d3_L1_p2": ("sod", 3, 1, 2, 4, {}, {}, True),
    "sf_sod_d2_L2_p1": ("sod", 2, 2, 1, 6, {"mode": "straightforward"}, {}, True),
}
BIG = {
    "bump_d3_L3_p3_cfg2": ("bump", 3, 3, 3, 20, {}, {}, False),
    "bump_d3_L3_p5_cfg3": ("bump", 3, 3, 5, 10, {}, {}, False),
    "bump_d3_L3_p7_cfg3": ("bump", 3, 3, 7, 10, {}, {}, False),
    "bump_d3_L3_p9_cfg3": ("bump", 3, 3, 9, 10, {}, {}, False),
    "bump_d3_L2_p5": ("bump", 3, 2, 5, 10, {}, {}, False),
    # round 2: reference-pinned state for the high-order kernels (p >= 6).  The 27^3 p=7 / p=9
    # runs stop one step before the reference's abort (step 7 / step 5), so the pre-abort state
    # and the Picard histogram are stored; the 9^3 random-Fourier runs are the cfg-5 state family
    "bump_d3_L3_p7_pre": ("bump", 3, 3, 7, 6, {}, {}, False),
    "bump_d3_L3_p9_pre": ("bump", 3, 3, 9, 4, {}, {}, False),
    "fourier_d3_L2_p9": ("fourier", 3, 2, 9, 5, {}, {}, False, 13),
    "fourier_d3_L2_p7": ("fourier", 3, 2, 7, 5, {}, {}, False, 13),
    "fourier_d3_L2_p6": ("fourier", 3, 2, 6, 4, {}, {}, False, 13),
}
SAMPLE_STRIDE = 97


def run_case(name, spec):
    from aderdg import (AdvectionSystem, Driver, EulerSystem, Kernels, NumericalError,
                        PredictorFailureError, TimeControl, build_grid, make_basis)
    scen, d, L, p, steps, dkw, tkw, full = spec[:8]
    stride = spec[8] if len(spec) > 8 else SAMPLE_STRIDE
    if scen.startswith("gauss"):
        from aderdg.cli import gaussian_profile
        Q0 = scenarios.build("gauss", d, L, p, **({"noise": 1e-2, "seed": 1} if scen == "gauss_noise" else {}))
        system = AdvectionSystem(d, scenarios.ADVECTION_VELOCITY[:d], profile=gaussian_profile)
    else:
        Q0 = scenarios.build(scen, d, L, p)
        system = EulerSystem(d)
    basis = make_basis(p)
    dkw = dict(dkw)
    mode = dkw.pop("mode", "fused")
    storage = "spacetime" if mode == "straightforward" else "hull"
    boundary = "outflow" if scen in scenarios.OUTFLOW else "periodic"
    grid = build_grid(d, L, p, system.m, boundary=boundary, storage=storage, budget_bytes=1 << 40)
    for c in grid.cells:
        c.Q[...] = Q0[c.index]
    kernels = Kernels(system, basis, grid, None, cfl=0.9)
    hist = {}
    orig_flux = system.flux
    calls = {"n": 0}

    def counting_flux(Q):   # predict calls flux once per Picard iteration + once at the end
        calls["n"] += 1
        return orig_flux(Q)

    system.flux = counting_flux
    orig_predict = kernels.predict

    def counting_predict(cell, dt):
        calls["n"] = 0
        out = orig_predict(cell, dt)
        k = calls["n"] - 1
        hist[k] = hist.get(k, 0) + 1
        return out

    kernels.predict = counting_predict
    tc = TimeControl(c_dt=0.99, **tkw)
    error = None
    t0 = time.time()
    try:
        driver = Driver(grid, kernels, tc, mode, **dkw)
        for _ in range(steps):
            driver.step()
    except (NumericalError, PredictorFailureError) as e:
        error = {"class": type(e).__name__, "message": str(e),
                 "cell": getattr(e, "cell_index", None)}
        driver = locals().get("driver")
    wall = time.time() - t0
    recs = driver.step_records if driver is not None else []
    rec_arr = np.array([[r["step"], r["T"], r["dt_old"], r["dt_new"], r["dt_adm"], r["reruns"]]
                        for r in recs], dtype=np.float64).reshape(-1, 6)
    Qf = np.stack([c.Q for c in grid.cells])
    out = {
        "records": rec_arr,
        "Q0_sum": np.array([np.sum(Q0), np.sum(np.abs(Q0))]),
        "Q_final_sum": np.sum(Qf.reshape(-1, Qf.shape[-1]), axis=0),
        "Q_final_absmax": np.max(np.abs(Qf.reshape(-1, Qf.shape[-1])), axis=0),
        "picard_keys": np.array(sorted(hist), dtype=np.int64),
        "picard_vals": np.array([hist[k] for k in sorted(hist)], dtype=np.int64),
        "meta": np.array(json.dumps({"scenario": scen, "system": system.name, "boundary": boundary,
                                     "d": d, "L": L, "p": p, "steps": steps,
                                     "driver_kwargs": dkw, "mode": mode, "tc_kwargs": tkw, "error": error,
                                     "wall_s": wall, "sweep_count": driver.sweep_count if driver else None,
                                     "rerun_count": driver.rerun_count if driver else None,
                                     "reruns_by_step": {str(k): v for k, v in
                                                        (driver.reruns_by_step.items() if driver else [])}})),
    }
    if error is None:
        if full:
            out["Q_final"] = Qf
        else:
            cells = np.arange(0, Qf.shape[0], stride)
            out["sample_cells"] = cells
            out["Q_sample"] = Qf[cells]
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: {wall:.1f}s steps={len(recs)} error={error}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*")
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()
    table = dict(SMALL)
    table.update(BIG)
    names = args.cases or (list(BIG) if args.big else list(SMALL))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    for n in names:
        run_case(n, table[n])


if __name__ == "__main__":
    main()
