"""Host-side API checks that need no GPU: argument validation mirrors the
reference (ConfigurationError before any device work), scenario determinism,
and the product never importing the oracle."""

import ast
import os

import numpy as np
import pytest

from conftest import REPO
from paper_1801_08682_b200 import (ConfigurationError, Driver, EulerSystem, Kernels,
                                   TimeControl, build_grid, device_bytes, make_basis,
                                   scenarios)
from paper_1801_08682_b200.errors import DomainError, ResourceBudgetError


def test_time_control_validation():
    # tests/test_scheduler.py:17-24 of the reference
    with pytest.raises(ConfigurationError):
        TimeControl(c_dt=0.0)
    with pytest.raises(ConfigurationError):
        TimeControl(c_dt=1.5)
    with pytest.raises(ConfigurationError):
        TimeControl(averaging="eager")


def test_build_grid_validation():
    with pytest.raises(ConfigurationError):
        build_grid(4, 1, 1, 6)
    with pytest.raises(ConfigurationError):
        build_grid(2, 0, 1, 4)
    with pytest.raises(ConfigurationError):
        build_grid(2, 5, 1, 4)
    with pytest.raises(ConfigurationError):
        build_grid(2, 1, 10, 4)
    with pytest.raises(ConfigurationError):
        build_grid(2, 1, 1, 4, boundary="reflective")
    assert build_grid(2, 1, 1, 4, boundary="outflow").boundary == "outflow"
    with pytest.raises(ResourceBudgetError):
        build_grid(3, 3, 3, 5, budget_bytes=1 << 20)
    g = build_grid(3, 2, 3, 5)
    assert g.Q.shape == (729, 4, 4, 4, 5) and g.h == 3.0 ** -2
    assert g.cells[10].multi_index == (0, 1, 1)
    g.cells[10].Q[...] = 7.0
    assert np.all(g.Q[10] == 7.0)


def test_euler_system_and_kernels_config():
    with pytest.raises(DomainError):
        EulerSystem(1)
    s = EulerSystem(2)
    assert (s.d, s.m, s.name) == (2, 4, "euler")
    g = build_grid(2, 1, 3, 4)
    k = Kernels(s, make_basis(3), g, None, cfl=0.9)
    w = k.basis.weights
    assert np.allclose(k.kvol, (k.basis.diff.T * w[None, :]) / w[:, None])
    assert k.picard_cap == 8
    with pytest.raises(ConfigurationError):
        Kernels(EulerSystem(3), make_basis(3), g, None)


@pytest.mark.parametrize("mode", ["shifted", "zigzag"])
def test_driver_modes_out_of_scope_fail_before_device(mode):
    g = build_grid(2, 1, 2, 4)
    k = Kernels(EulerSystem(2), make_basis(2), g, None)
    with pytest.raises(ConfigurationError):
        Driver(g, k, TimeControl(), mode)


def test_driver_rejects_limiter_and_bad_traversal():
    g = build_grid(2, 1, 2, 4)
    k = Kernels(EulerSystem(2), make_basis(2), g, None)
    with pytest.raises(ConfigurationError):
        Driver(g, k, TimeControl(), "fused", limiter=object())
    with pytest.raises(ConfigurationError):
        Driver(g, k, TimeControl(), "fused", traversal="zigzag")
    with pytest.raises(ConfigurationError):
        Driver(g, k, TimeControl(), "fused", traversal=np.array([0, 0, 1, 2, 3, 4, 5, 6, 7]))


def test_scenarios_deterministic_and_physical():
    a = scenarios.build("bump", 3, 1, 3, seed=0)
    b = scenarios.build("bump", 3, 1, 3, seed=0)
    c = scenarios.build("bump", 3, 1, 3, seed=1)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    rho = a[..., 0]
    p = 0.4 * (a[..., -1] - 0.5 * np.sum(a[..., 1:4] ** 2, axis=-1) / rho)
    assert np.allclose(p, 1.0, atol=1e-12)
    f = scenarios.build("fourier", 3, 1, 2, seed=0)
    assert f.shape == (27, 3, 3, 3, 5) and np.all(f[..., 0] > 0.7)


def test_device_bytes_fit_one_b200():
    # every BASELINE configuration fits one 180 GB B200 (cfg 5: 81^3 at p = 9)
    assert device_bytes(3, 4, 9) < 150e9
    assert device_bytes(3, 3, 3) < 1e9


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_1801_08682_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            tree = ast.parse(open(os.path.join(pkg, fn)).read())
            for node in ast.walk(tree):
                if isinstance(node, (ast.Import, ast.ImportFrom)):
                    names = [a.name for a in node.names] + [getattr(node, "module", "") or ""]
                    assert not any("oracle" in n for n in names), fn


def test_limiter_mode_restriction():
    """reference tests/test_limiter.py:170-176 (raised before any device work)."""
    from paper_1801_08682_b200 import (ConfigurationError, Driver, EulerSystem, Kernels, SubcellLimiter,
                                       TimeControl, build_grid, make_basis, scenarios)
    grid = build_grid(2, 1, 2, 4)
    grid.Q[...] = scenarios.build("wave", 2, 1, 2)
    basis = make_basis(2)
    lim = SubcellLimiter(EulerSystem(2), basis, grid)
    with pytest.raises(ConfigurationError, match="straightforward mode only"):
        Driver(grid, Kernels(EulerSystem(2), basis, grid, None), TimeControl(), "fused", limiter=lim)


def test_limiter_operators_match_reference_construction():
    """SubcellLimiter operators (src/limiter.py:26-34,96-108) against the oracle's restatement."""
    import limiter_oracle as LO
    import aderdg_oracle as O
    from paper_1801_08682_b200 import EulerSystem, SubcellLimiter, build_grid, make_basis
    for d, p in ((2, 0), (2, 3), (3, 5), (3, 9)):
        grid = build_grid(d, 1, p, d + 2)
        lim = SubcellLimiter(EulerSystem(d), make_basis(p), grid)
        ora = LO.OracleLimiter(O.OracleKernels(d, p, 1))
        P, R, nearest, sample = lim.device_arrays()
        assert np.array_equal(P, ora.P) and np.array_equal(R, ora.R)
        assert np.array_equal(nearest, ora.nearest) and np.array_equal(sample, ora.sample)
        assert lim.h_sub == ora.h_sub
