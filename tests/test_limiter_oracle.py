"""CPU checks of the subcell-limiter oracle (oracle/limiter_oracle.py).

* pinned to the reference: golden runs of ``Driver(..., "straightforward",
  limiter=SubcellLimiter(...))`` written by ``tests/golden/make_limiter_golden.py``
  (final state, per-step troubled counts and dt log, final troubled flags);
* the reference's own limiter known-answer tests restated on the oracle
  (``tests/test_limiter.py:17-167`` of the reference).
"""

import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, REPO)

import aderdg_oracle as O  # noqa: E402
import limiter_oracle as LO  # noqa: E402
from paper_1801_08682_b200 import scenarios  # noqa: E402

GOLD = os.path.join(HERE, "golden")
CASES = sorted(f[4:-4] for f in os.listdir(GOLD) if f.startswith("lim_") and f.endswith(".npz"))


def load_case(name):
    g = np.load(os.path.join(GOLD, f"lim_{name}.npz"))
    meta = json.loads(str(g["meta"]))
    Q0 = scenarios.build(meta["scenario"], meta["d"], meta["L"], meta["p"], **meta["scenario_kwargs"])
    assert np.allclose([np.sum(Q0), np.sum(np.abs(Q0))], g["Q0_sum"], rtol=1e-14, atol=0)
    return g, meta, Q0


def run_oracle(meta, Q0, order=None):
    drv = LO.LimitedStraightforwardDriver(Q0.copy(), meta["d"], meta["p"], meta["L"], order=order,
                                          boundary=meta.get("boundary", "periodic"), **meta["tc_kwargs"])
    with np.errstate(all="ignore"):
        drv.run(meta["steps"])
    return drv


def test_cases_present():
    assert len(CASES) >= 6


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_limiter(name):
    g, meta, Q0 = load_case(name)
    assert meta["error"] is None
    drv = run_oracle(meta, Q0, g["order"] if "order" in g else None)
    ref = g["Q_final"]
    assert np.max(np.abs(drv.Q - ref)) <= 1e-12 * np.max(np.abs(ref))
    rec = np.array([[r["step"], r["T"], r["dt_old"], r["dt_new"], r["dt_adm"], r["troubled"]]
                    for r in drv.step_records])
    assert np.array_equal(rec[:, 5], g["records"][:, 5])         # troubled cells per step
    assert np.allclose(rec[:, 1:5], g["records"][:, 1:5], rtol=1e-12, atol=0)
    assert np.array_equal(drv.troubled, g["troubled_final"])
    assert g["records"][:, 5].sum() > 0                           # the limiter really acted


def _lim(d=2, p=3, L=1):
    k = O.OracleKernels(d, p, L)
    return k, LO.OracleLimiter(k)


def test_subcell_average_matrix_exact_on_monomials():
    """reference tests/test_limiter.py:17-27."""
    b = O.make_basis(3)
    P = LO.subcell_average_matrix(b)
    ns = 2 * b.p + 1
    edges = np.arange(ns + 1) / ns
    for k in range(b.n):
        want = (edges[1:] ** (k + 1) - edges[:-1] ** (k + 1)) / ((k + 1) * (edges[1:] - edges[:-1]))
        assert np.allclose(P @ b.nodes ** k, want, atol=1e-13)
    assert np.allclose(P.sum(axis=1), 1.0, atol=1e-13)


def test_projection_reconstruction_round_trip():
    """reference tests/test_limiter.py:38-52: polynomials of degree <= p survive."""
    k, lim = _lim(p=3)
    x = scenarios.node_coordinates(2, 1, 3)[4]
    Q = scenarios.smooth_density_wave(2, 1, 3)[4]
    Q[..., 0] = 1.0 + x[..., 0] ** 2 - 0.3 * x[..., 0] * x[..., 1]
    patch = lim.project(Q)
    assert patch.shape == (7, 7, 4)
    Qr, ok = lim.reconstruct(patch)
    assert ok and np.max(np.abs(Qr - Q)) < 1e-12


def test_reconstruction_preserves_patch_mean():
    """reference tests/test_limiter.py:55-62."""
    k, lim = _lim(p=2)
    patch = 1.0 + 0.1 * np.random.default_rng(5).normal(size=(5, 5, 4))
    patch[..., -1] += 5.0
    Q, _ = lim.reconstruct(patch)
    assert np.allclose(np.sum(lim.mean_weights * Q, axis=(0, 1)), patch.mean(axis=(0, 1)), atol=1e-13)


def test_fv_step_fixed_point_and_conservation():
    """reference tests/test_limiter.py:74-85."""
    pde = O.EulerPDE(2)
    states = np.tile([1.0, 0.4, -0.2, 2.5], (6, 6, 1))
    assert np.max(np.abs(LO.rusanov_fv_step(states, 0.1, 1e-3, pde) - states)) < 1e-14
    states = states + 0.05 * np.random.default_rng(7).normal(size=states.shape)
    out = LO.rusanov_fv_step(states, 0.1, 1e-3, pde)
    assert np.allclose(out.sum(axis=(0, 1)), states.sum(axis=(0, 1)), atol=1e-12)


def test_fv_step_enforces_cfl():
    """reference tests/test_limiter.py:88-92."""
    pde = O.AdvectionPDE(2, (1.0, 0.0))
    with pytest.raises(O.OracleError):
        LO.rusanov_fv_step(np.ones((4, 4, 1)), 0.1, 0.1, pde)


def test_fv_step_matches_degree_zero_pipeline():
    """reference tests/test_limiter.py:95-114 / test_acceptance.py:172-190: at
    p = 0 the predictor-corrector pipeline is the first-order Godunov scheme."""
    Q0 = scenarios.smooth_density_wave(2, 2, 0)
    dt = 2e-3
    drv = O.StraightforwardDriver(Q0.copy(), 2, 0, 2, forced_dt=dt)
    drv.run(20)
    block = Q0[:, 0, 0].reshape(9, 9, 4)
    pde = O.EulerPDE(2)
    for _ in range(20):
        block = LO.rusanov_fv_step(block, 3.0 ** -2, dt, pde)
    assert np.max(np.abs(drv.Q[:, 0, 0].reshape(9, 9, 4) - block)) <= 1e-13


def test_detection_accepts_smooth_and_flags_overshoot():
    """reference tests/test_limiter.py:117-127."""
    k, lim = _lim(p=2, L=1)
    Q = scenarios.smooth_density_wave(2, 1, 2)
    rank = np.arange(Q.shape[0])
    assert not lim.detect(Q, Q, Q, rank)[4]
    Q2 = Q.copy()
    Q2[4, 0, 0, 0] += 0.5
    assert lim.detect(Q2, Q, Q, rank)[4]
    Q2[4, ..., 0] = -1.0
    assert lim.detect(Q2, Q, Q, rank)[4]


def test_cell_mean_conserved_through_limiting_pipeline():
    """reference tests/test_limiter.py:154-167."""
    k, lim = _lim(p=3)
    Q = scenarios.smooth_density_wave(2, 1, 3)[4]
    patch = lim.project(Q)
    mean0 = patch.mean(axis=(0, 1))
    for _ in range(5):
        patch = LO.rusanov_fv_step(patch, lim.h_sub, 1e-4, lim.pde)
    Qr, ok = lim.reconstruct(patch)
    assert ok
    mean1 = np.sum(lim.mean_weights * Qr, axis=(0, 1))
    assert np.max(np.abs(mean1 - patch.mean(axis=(0, 1)))) < 1e-13
    assert np.max(np.abs(mean1 - mean0) / np.abs(mean0)) < 1e-11
