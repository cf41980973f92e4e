"""Pin the CPU oracle (oracle/aderdg_oracle.py) against golden vectors that the
reference implementation itself produced (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import aderdg_oracle as O
from conftest import golden_boundary, golden_names, golden_problem, load_golden, rel_linf

FAST = [n for n in golden_names() if n in (
    "bump_d2_L2_p3", "bump_d2_L1_p0", "bump_d2_L2_p1", "bump_d2_L1_p9", "bump_d2_L2_p6",
    "bump_d3_L1_p3", "bump_d3_L1_p2", "bump_d3_L1_p5", "fourier_d3_L1_p4",
    "wave_d2_L1_p2_spike", "wave_d2_L1_p3_inject", "wave_d2_L2_p3_forced",
    "wave_d3_L1_p2_creeping", "uniform_d2_L1_p2", "bump_d2_L3_p3_cfg1")
        or n.startswith("sf_") or n.startswith("adv_") or n.startswith("sod_")]


def run_oracle(meta):
    Q0, vel = golden_problem(meta)
    dkw = dict(meta["driver_kwargs"])
    if vel is not None:
        dkw["velocity"] = vel
    tkw = dict(meta["tc_kwargs"])
    cls = O.StraightforwardDriver if meta.get("mode", "fused") == "straightforward" else O.FusedDriver
    drv = cls(Q0.copy(), meta["d"], meta["p"], meta["L"], boundary=golden_boundary(meta), **dkw, **tkw)
    err = None
    try:
        for _ in range(meta["steps"]):
            drv.step()
    except O.OracleError as e:
        err = e
    return drv, err, Q0


@pytest.mark.parametrize("name", FAST)
def test_oracle_matches_reference_golden(name):
    g = load_golden(name)
    meta = g["meta"]
    drv, err, Q0 = run_oracle(meta)
    assert np.allclose([np.sum(Q0), np.sum(np.abs(Q0))], g["Q0_sum"], rtol=1e-15, atol=0)
    if meta["error"] is not None:
        assert err is not None and err.kind == meta["error"]["class"]
        assert str(err) == f"{err.kind}: {meta['error']['message']}"
        if meta["error"]["cell"] is not None:
            assert err.cell_index == meta["error"]["cell"]
        return
    assert err is None
    recs = np.array([[r["step"], r["T"], r["dt_old"], r["dt_new"], r["dt_adm"], r["reruns"]]
                     for r in drv.step_records])
    ref = g["records"]
    assert recs.shape == ref.shape
    assert np.array_equal(recs[:, 0], ref[:, 0])
    assert np.array_equal(recs[:, 5], ref[:, 5]), "rerun steps differ"
    assert np.max(np.abs(recs[:, 1:5] - ref[:, 1:5]) / np.abs(ref[:, 1:5]).clip(1e-300)) < 1e-12
    assert drv.sweep_count == meta["sweep_count"]
    assert drv.rerun_count == meta["rerun_count"]
    if "Q_final" in g:
        assert rel_linf(drv.Q, g["Q_final"]) < 1e-12
    else:
        assert rel_linf(drv.Q[g["sample_cells"]], g["Q_sample"]) < 1e-12
    hist = dict(drv.k.picard_hist)
    ref_hist = dict(zip(g["picard_keys"].tolist(), g["picard_vals"].tolist()))
    assert hist == ref_hist
