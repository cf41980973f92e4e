"""Host logic of the batch front end (paper_1801_08682_b200/cli.py, metrics.py)
against the reference's own CLI behaviour (tests/test_cli.py of the reference)
and its artifacts (tests/golden/cli/*, made by tests/golden/make_cli_golden.py).
No GPU needed: everything here stops before a Driver is built, or replays the
closed-form ledger."""

import csv
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1801_08682_b200 import ConfigurationError, metrics
from paper_1801_08682_b200.cli import (METRIC_COLUMNS, RunConfig, main, scenario,
                                       setup_run)

CLI = os.path.join(GOLDEN, "cli")
RUN_CASES = sorted(c for c in os.listdir(CLI) if os.path.exists(os.path.join(CLI, c, "metrics.csv")))


def read_metrics(path):
    with open(path, newline="") as fh:
        return list(csv.DictReader(fh))


def test_scenario_catalogue():
    system, init, boundary = scenario("uniform", 2)
    assert boundary == "periodic"
    assert np.allclose(init(np.zeros((1, 2))), [[1.0, 0.0, 0.0, 2.5]])
    system, init, boundary = scenario("sod", 2)
    assert boundary == "outflow"
    states = init(np.array([[0.25, 0.5], [0.75, 0.5]]))
    assert np.allclose(states, [[1.0, 0.0, 0.0, 2.5], [0.125, 0.0, 0.0, 0.25]])
    system, init, boundary = scenario("gaussian-advect", 3)
    assert system.name == "advection" and system.m == 1
    assert np.allclose(system.velocity, (1.0, 0.5, 0.25))
    assert init(np.full((1, 3), 0.5))[0, 0] == pytest.approx(1.0)
    with pytest.raises(ConfigurationError):
        scenario("blast-wave", 2)


def test_config_file_parsing(tmp_path):
    f = tmp_path / "case.cfg"
    f.write_text("# euler smoke case\nscenario = smooth-density-wave\nmode = shifted   # pipelined\n"
                 "steps = 7\np = 4\nlimiter = no\nforced_dt = 1e-4\n\n")
    cfg = RunConfig.from_file(f)
    assert (cfg.mode, cfg.steps, cfg.p, cfg.limiter, cfg.forced_dt) == ("shifted", 7, 4, False, 1e-4)
    f.write_text("colour = blue\n")
    with pytest.raises(ConfigurationError):
        RunConfig.from_file(f)
    f.write_text("just a line without an equals sign\n")
    with pytest.raises(ConfigurationError):
        RunConfig.from_file(f)
    with pytest.raises(ConfigurationError):
        RunConfig(scenario="warp-drive").validate()
    with pytest.raises(ConfigurationError):
        RunConfig(p=12).validate()


@pytest.mark.parametrize("kw,msg", [
    (dict(mode="shifted"), "shifted"),
    (dict(limiter=True), "straightforward mode only"),
    (dict(trace=True), "trace"),
])
def test_outside_gpu_path_is_a_configuration_error(kw, msg):
    with pytest.raises(ConfigurationError) as e:
        setup_run(RunConfig(**kw))
    assert msg in str(e.value)


def test_main_exit_code_for_bad_config(tmp_path, capsys):
    bad = tmp_path / "bad.cfg"
    bad.write_text("scenario = blast-wave\n")
    assert main(["run", "--config", str(bad), "--out", str(tmp_path / "bad")]) == 2
    assert "configuration error" in capsys.readouterr().err


@pytest.mark.parametrize("case", RUN_CASES)
def test_closed_form_ledger_matches_reference_metrics(case):
    """Replaying the reference's rerun decisions through metrics.record_step gives
    the reference's integer ledger columns and run.json audit figures."""
    kw = json.load(open(os.path.join(CLI, case, "case.json")))
    cfg = RunConfig(**kw)
    system, _, boundary = scenario(cfg.scenario, cfg.d)
    rows = read_metrics(os.path.join(CLI, case, "metrics.csv"))
    led = metrics.AccessLedger(cfg.mode, cfg.d, cfg.p, system.m)
    K = 3 ** cfg.L
    cells = K ** cfg.d
    faces = cfg.d * cells if boundary == "periodic" else cfg.d * (K + 1) * K ** (cfg.d - 1)
    for row in rows:
        rec = metrics.record_step(led, cfg.mode, int(row["step"]), int(row["reruns"]), cells,
                                  faces, int(row["troubled"]))
        for col in METRIC_COLUMNS:
            if col in ("step", "T", "dt_old", "dt_new", "dt_adm", "reruns", "troubled", "wall_time"):
                continue
            assert float(row[col]) == float(rec.get(col, 0)), (case, row["step"], col)
    man = json.load(open(os.path.join(CLI, case, "run.json")))
    audit = metrics.single_touch_audit(led, cells, len(rows))
    assert audit["amortised"] == man["q_reads_per_cell_step"]
    storage = "spacetime" if cfg.mode == "straightforward" else "hull"
    assert metrics.estimate_persistent_doubles(cfg.d, cfg.L, cfg.p, system.m, boundary,
                                               storage) == man["persistent_doubles"]


def test_traffic_models():
    # src/metrics.py:217-230 closed forms and the fused/straightforward footprint ratio
    assert metrics.traffic_model("straightforward", 3, 3, 5) == 58 * 5 * 64
    assert metrics.traffic_model("fused", 3, 3, 5, 1.0) == 51 * 5 * 64
    assert metrics.footprint_ratio(3, 3) == metrics.Fraction(20, 35)
    assert metrics.rerun_upper_bound(3.0, 1.5, 1.2, 0.9) == 2.0


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not present")
@pytest.mark.parametrize("d,L,p", [(2, 1, 2), (2, 2, 3), (3, 1, 4)])
def test_l2_error_matches_reference(d, L, p):
    """The convergence study's L2 error (host post-processing) against the reference's
    l2_error (src/cli.py:256-275) on a perturbed advection state."""
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from aderdg import cli as rcli
    from aderdg.basis import make_basis as rbasis
    from aderdg.mesh import build_grid as rgrid
    from aderdg.pde import AdvectionSystem as RAdv
    from paper_1801_08682_b200 import AdvectionSystem
    from paper_1801_08682_b200.cli import cell_node_coordinates, gaussian_profile, l2_error
    rng = np.random.default_rng(4)
    basis = rbasis(p)
    x = cell_node_coordinates(d, L, basis.nodes)
    Q = gaussian_profile(x)[..., None] + 1e-3 * rng.standard_normal(x.shape[:-1] + (1,))
    ours = l2_error(Q, d, L, p, AdvectionSystem(d, (1.0, 0.5, 0.25)[:d], profile=gaussian_profile), 0.03)
    grid = rgrid(d, L, p, 1, budget_bytes=1 << 40)
    for c in grid.cells:
        c.Q[...] = Q[c.index]
    ref = rcli.l2_error(grid, basis, RAdv(d, (1.0, 0.5, 0.25)[:d], profile=rcli.gaussian_profile), 0.03)
    assert abs(ours - ref) <= 1e-12 * ref
