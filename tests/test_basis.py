"""Host-side operators: bitwise equal to the reference's make_basis (via the
pinned oracle restatement) and the reference's basis KATs
(tests/test_basis.py:10-74 of the reference)."""

import numpy as np
import pytest

import aderdg_oracle as O
from paper_1801_08682_b200 import ConfigurationError, make_basis


@pytest.mark.parametrize("p", range(10))
def test_operators_bitwise_equal_oracle(p):
    a, b = make_basis(p), O.make_basis(p)
    for f in ("nodes", "weights", "diff", "left", "right", "integ"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


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


def test_order_validation():
    with pytest.raises(ConfigurationError):
        make_basis(10)
    with pytest.raises(ConfigurationError):
        make_basis(-1)
