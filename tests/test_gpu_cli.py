"""The batch front end on the GPU against the reference's own artifacts
(tests/golden/cli/*, written by the reference's run_simulation /
convergence_study), plus the reference's convergence acceptance bars
(tests/test_acceptance.py:135-160 of the reference) for the AdvectionSystem
plug-in of the sweep kernel."""

import csv
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1801_08682_b200.cli import RunConfig, convergence_study, main, run_simulation

pytestmark = pytest.mark.gpu
TOL = 1e-10
CLI = os.path.join(GOLDEN, "cli")
RUN_CASES = sorted(c for c in os.listdir(CLI) if os.path.exists(os.path.join(CLI, c, "metrics.csv")))
FLOAT_COLS = ("T", "dt_old", "dt_new", "dt_adm")


def read_csv(path):
    with open(path, newline="") as fh:
        return list(csv.DictReader(fh))


def solution(path):
    rows = read_csv(path)
    return np.array([[float(v) for k, v in r.items() if k != "cell"] for r in rows])


@pytest.mark.parametrize("case", RUN_CASES)
def test_run_artifacts_match_reference(cuda_ok, tmp_path, case):
    kw = json.load(open(os.path.join(CLI, case, "case.json")))
    out = run_simulation(RunConfig(out=str(tmp_path / case), **kw))
    ref_rows = read_csv(os.path.join(CLI, case, "metrics.csv"))
    rows = read_csv(out / "metrics.csv")
    assert list(rows[0].keys()) == list(ref_rows[0].keys())
    assert len(rows) == len(ref_rows)
    for r, g in zip(rows, ref_rows):
        for k in g:
            if k == "wall_time":
                continue
            if k in FLOAT_COLS:
                assert abs(float(r[k]) - float(g[k])) <= TOL * abs(float(g[k])), (case, k)
            else:
                assert r[k] == g[k], (case, r["step"], k)
    S, G = solution(out / "solution_final.csv"), solution(os.path.join(CLI, case, "solution_final.csv"))
    assert S.shape == G.shape
    assert np.max(np.abs(S - G)) <= TOL * np.max(np.abs(G))
    man = json.loads((out / "run.json").read_text())
    ref = json.load(open(os.path.join(CLI, case, "run.json")))
    assert abs(man.pop("final_time") - ref.pop("final_time")) <= TOL * abs(ref["config"]["final_time"] or 1.0)
    man["config"].pop("out")
    ref["config"].pop("out")
    assert man == ref


def test_runs_are_bytewise_deterministic(cuda_ok, tmp_path):
    outs = [run_simulation(RunConfig(scenario="smooth-density-wave", mode="fused", steps=4,
                                     out=str(tmp_path / t))) for t in "ab"]
    assert (outs[0] / "solution_final.csv").read_bytes() == (outs[1] / "solution_final.csv").read_bytes()

    def strip(o):
        return [{k: v for k, v in r.items() if k != "wall_time"} for r in read_csv(o / "metrics.csv")]
    assert strip(outs[0]) == strip(outs[1])


def test_main_convergence_subcommand_matches_reference(cuda_ok, tmp_path):
    case = json.load(open(os.path.join(CLI, "conv_p2", "case.json")))
    assert main(["convergence", "--p", "2", "--levels", ",".join(map(str, case["levels"])),
                 "--final-time", str(case["final_time"]), "--out", str(tmp_path / "conv")]) == 0
    rows = read_csv(tmp_path / "conv" / "convergence.csv")
    ref = read_csv(os.path.join(CLI, "conv_p2", "convergence.csv"))
    for r, g in zip(rows, ref):
        assert abs(float(r["error"]) - float(g["error"])) <= 1e-8 * float(g["error"])
    assert float(rows[1]["order"]) > 2.0


@pytest.mark.parametrize("p,levels,lo,hi", [(2, (1, 2, 3), 2.5, None), (3, (1, 2, 3), 3.5, None),
                                            (0, (2, 3, 4), 0.8, 1.2)])
def test_convergence_orders(cuda_ok, p, levels, lo, hi):
    rows = convergence_study(RunConfig(scenario="gaussian-advect", d=2, p=p), levels, final_time=0.05)
    order = rows[-1]["order"]
    assert order >= lo
    if hi is not None:
        assert order <= hi


def test_convergence_3d_high_order(cuda_ok):
    """The advection plug-in at d = 3, p = 5 (beyond the reference's 2-D study)."""
    rows = convergence_study(RunConfig(scenario="gaussian-advect", d=3, p=5), (1, 2), final_time=0.02)
    assert rows[-1]["order"] >= 5.0
