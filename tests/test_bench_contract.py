"""The driver's bench contract: one JSON line with the keys the round-end harness reads.
The reference arm runs on CPU (oracle port); our arm needs a GPU."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def run_bench(*args):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True,
                         text=True, timeout=900, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "cfg1", "--steps", "2")
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["unit"] == "DoF-updates/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["name"] == "cfg1" and "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and "nproc" in cb["sample"]
    assert [r["label"] for r in cb["rows"]][0] == "1 pinned core"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_gpus_flag_needs_that_many_devices():
    import torch
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", str(max(2, have + 1))],
                         capture_output=True, text=True, timeout=300, cwd=REPO)
    assert out.returncode == 2 and "visible GPUs" in out.stderr


@pytest.mark.gpu
def test_our_arm_line(cuda_ok):
    d = run_bench("--config", "cfg1", "--no-cpu-baseline")
    assert (BASE_KEYS | {"roofline", "gpu_launches", "clocks"}) <= set(d)
    assert d["n_gpus"] == 1 and d["dtype"] == "f64" and d["data"] == "synthetic" and d["warmup"] >= 3
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "TFLOP/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12 and 0 < r["frac"] < 1
    assert r["kernel_ms_per_step"] <= d["ms_per_step"] * (1 + 1e-9)
    # cfg 1 runs each timed segment as one cooperative multi-step launch
    assert d["gpu_launches"] == d["run"]["episodes"] >= 1
    assert r["kernel_ms_per_step"] == pytest.approx(d["ms_per_step"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 8 * d["config"]["dof"]
    assert e["value"] < d["value"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
