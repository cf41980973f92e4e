"""Host-side operators: the committed table (paper_1801_08682_b200/data/operators.npz)
is bitwise the reference's make_basis / SubcellLimiter operators (checked against the
reference itself where it is importable, and always against the pinned oracle
restatement), and meets the reference's basis KATs (tests/test_basis.py:10-74 of the
reference)."""

import os
import sys

import numpy as np
import pytest

import aderdg_oracle as O
from paper_1801_08682_b200 import ConfigurationError, make_basis
from paper_1801_08682_b200.basis import operator_table, quadrature6, subcell_operators

REF = "/root/reference/pkg/src"


def _reference():
    if not os.path.isdir(REF):
        return None
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import aderdg.basis as rb
    import aderdg.limiter as rl
    import aderdg.mesh as rm
    import aderdg.pde as rp
    return rb, rl, rm, rp


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
@pytest.mark.parametrize("p", range(10))
def test_table_bitwise_equal_reference(p):
    rb, rl, rm, rp = _reference()
    ref = rb.make_basis(p)
    ours = make_basis(p)
    for f in ("nodes", "weights", "diff", "left", "right", "integ"):
        assert np.array_equal(getattr(ours, f), getattr(ref, f)), f
    lim = rl.SubcellLimiter(rp.EulerSystem(2), ref, rm.build_grid(2, 1, p, 4, budget_bytes=1 << 40))
    P, R = subcell_operators(p)
    assert np.array_equal(P, lim.P) and np.array_equal(R, lim.R)
    x6, w6, E6 = quadrature6(p)
    assert np.array_equal(E6, rb.lagrange_eval(ref.nodes, x6))
    assert np.array_equal(x6, rb.make_basis(5).nodes) and np.array_equal(w6, rb.make_basis(5).weights)


@pytest.mark.parametrize("p", range(10))
def test_operators_bitwise_equal_oracle(p):
    a, b = make_basis(p), O.make_basis(p)
    for f in ("nodes", "weights", "diff", "left", "right", "integ"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_table_is_read_only():
    tab = operator_table()
    with pytest.raises(ValueError):
        tab["p3_diff"][0, 0] = 1.0


@pytest.mark.parametrize("p", range(10))
def test_gauss_legendre_matches_numpy(p):
    b = make_basis(p)
    x, w = np.polynomial.legendre.leggauss(p + 1)
    assert np.allclose(b.nodes, 0.5 * (x + 1.0), atol=1e-14)
    assert np.allclose(b.weights, 0.5 * w, atol=1e-14)


@pytest.mark.parametrize("p", range(1, 10))
def test_diff_exact_on_monomials_and_rows_sum_to_zero(p):
    b = make_basis(p)
    for k in range(p + 1):
        assert np.allclose(b.diff @ b.nodes ** k, k * b.nodes ** max(k - 1, 0) * (k > 0), atol=1e-9)
    assert np.allclose(b.diff.sum(axis=1), 0.0, atol=1e-12)


@pytest.mark.parametrize("p", range(10))
def test_integ_and_traces_exact(p):
    b = make_basis(p)
    for k in range(p + 1):
        assert np.allclose(b.integ @ b.nodes ** k, b.nodes ** (k + 1) / (k + 1), atol=1e-12)
        assert np.isclose(b.left @ b.nodes ** k, 0.0 ** k, atol=1e-12)
        assert np.isclose(b.right @ b.nodes ** k, 1.0, atol=1e-11)


@pytest.mark.parametrize("p", range(10))
def test_subcell_and_quadrature_operators_exact(p):
    b = make_basis(p)
    P, R = subcell_operators(p)
    ns = 2 * p + 1
    # the subcell averages of a constant are that constant; R lifts P back (least squares)
    assert np.allclose(P.sum(axis=1), 1.0, atol=1e-12)
    assert np.allclose(R @ P, np.eye(p + 1), atol=1e-9)
    x6, w6, E6 = quadrature6(p)
    for k in range(p + 1):
        assert np.allclose(E6 @ b.nodes ** k, x6 ** k, atol=1e-11)
        # average of x^k over subcell s
        s = np.arange(ns)
        exact = ((s + 1.0) ** (k + 1) - s ** (k + 1.0)) / ((k + 1) * ns ** k)
        assert np.allclose(P @ b.nodes ** k, exact, atol=1e-11)


def test_order_validation():
    with pytest.raises(ConfigurationError):
        make_basis(10)
    with pytest.raises(ConfigurationError):
        make_basis(-1)
