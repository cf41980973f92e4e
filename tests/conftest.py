import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running case")


def golden_names():
    """Driver goldens of make_golden.py (the limiter's lim_* goldens have their own tests)."""
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and not f.startswith("lim_"))


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    out = {k: z[k] for k in z.files}
    out["meta"] = json.loads(str(out["meta"]))
    return out


def golden_problem(meta):
    """Initial state and PDE of a golden case: (Q0, velocity or None).  The
    ``gauss*`` scenarios are AdvectionSystem(d, (1.0, 0.5, 0.25)[:d]) runs
    (src/cli.py:31,139-142), everything else EulerSystem(d)."""
    from paper_1801_08682_b200 import scenarios
    d, L, p = meta["d"], meta["L"], meta["p"]
    scen = meta["scenario"]
    if scen.startswith("gauss"):
        kw = {"noise": 1e-2, "seed": 1} if scen == "gauss_noise" else {}
        return scenarios.build("gauss", d, L, p, **kw), scenarios.ADVECTION_VELOCITY[:d]
    return scenarios.build(scen, d, L, p), None


def golden_boundary(meta):
    """Grid boundary of a golden case (the sod scenario runs with outflow, src/cli.py:155)."""
    return meta.get("boundary", "periodic")


def make_system(d, velocity):
    from paper_1801_08682_b200 import AdvectionSystem, EulerSystem
    return EulerSystem(d) if velocity is None else AdvectionSystem(d, velocity)


def rel_linf(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
