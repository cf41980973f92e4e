"""Seeded initial states of the BASELINE configurations (host-side input builders).

The reference has no random scenarios (``src/cli.py:4-5``), so the BASELINE
states are defined here once and fed, as the same host array, to the GPU path
and to the CPU oracle.  Conventions follow the reference:

* node coordinates ``x = (i_cell + nodes) * h`` per axis, ``meshgrid(...,
  indexing="ij")`` (``src/cli.py:160-166``), ``h = 3**-L`` (``src/mesh.py:71``);
* cell order = C-order ravel of the cell multi-index (``src/mesh.py:191-193``);
* conserved variables ``(rho, j_1..j_d, E)`` with ``E = p/(1.4-1.0) + rho|u|^2/2``
  (``src/pde.py:27-32`` uses ``GAMMA - 1.0``).

Array layout returned: ``(n_cells,) + (p+1,)*d + (d+2,)`` float64, i.e. the
reference's ``stack([c.Q for c in grid.cells])`` (``tests/conftest.py:77-79``).
"""

import numpy as np

from .basis import make_basis

GAMMA = 1.4


def node_coordinates(d, L, p):
    """(n_cells,) + (n,)*d + (d,) physical node coordinates."""
    b = make_basis(p)
    K = 3 ** L
    h = 3.0 ** (-L)
    idx = np.stack(np.unravel_index(np.arange(K ** d), (K,) * d), axis=-1)  # (C, d)
    axes = [(idx[:, a][:, None] + b.nodes[None, :]) * h for a in range(d)]  # (C, n)
    grids = []
    for a in range(d):
        shape = [K ** d] + [1] * d
        shape[1 + a] = b.n
        grids.append(np.broadcast_to(axes[a].reshape(shape), (K ** d,) + (b.n,) * d))
    return np.stack(grids, axis=-1)


def conserved(rho, u, p):
    """(rho, u[..., d], p) -> conserved state with component axis last."""
    d = u.shape[-1]
    Q = np.empty(rho.shape + (d + 2,))
    Q[..., 0] = rho
    for a in range(d):
        Q[..., 1 + a] = rho * u[..., a]
    Q[..., -1] = p / (GAMMA - 1.0) + 0.5 * rho * np.sum(u * u, axis=-1)
    return Q


def gaussian_bump_noise(d, L, p, seed=0, noise=1e-3, velocity=None):
    """BASELINE configs 1-4: rho = 1 + 0.2 exp(-|x-0.5|^2/0.01) + U(-noise, noise),
    u = (0.5, 0.3[, 0.2]), p = 1.  The noise is drawn once per node with
    ``default_rng(seed).uniform(-noise, noise, size=(n_cells,)+(n,)*d)``."""
    x = node_coordinates(d, L, p)
    n_cells = x.shape[0]
    n = p + 1
    r2 = np.sum((x - 0.5) ** 2, axis=-1)
    rho = 1.0 + 0.2 * np.exp(-r2 / 0.01)
    if noise:
        rng = np.random.default_rng(seed)
        rho = rho + rng.uniform(-noise, noise, size=(n_cells,) + (n,) * d)
    if velocity is None:
        velocity = (0.5, 0.3, 0.2)[:d]
    u = np.broadcast_to(np.asarray(velocity, dtype=float), rho.shape + (d,))
    return conserved(rho, u, np.ones_like(rho))


def random_fourier(d, L, p, seed=0, modes=4, rho_amp=0.05, u_amp=0.2):
    """BASELINE config 5: rho = 1 + 0.05 sum_k sin(2 pi kappa_k.x + phi_k),
    u_a = 0.2 sum_k sin(2 pi kappa'_{a,k}.x + phi'_{a,k}), p = 1, integer wave
    vectors in {1,2,3}^d.  Draw order from ``default_rng(seed)``: for each of
    the ``modes`` density modes kappa (integers(1, 4, d)) then phi
    (uniform(0, 2pi)); then for each axis a and mode k, kappa' then phi'."""
    x = node_coordinates(d, L, p)
    rng = np.random.default_rng(seed)
    rho = np.ones(x.shape[:-1])
    for _ in range(modes):
        kappa = rng.integers(1, 4, size=d)
        phi = rng.uniform(0.0, 2.0 * np.pi)
        rho = rho + rho_amp * np.sin(2.0 * np.pi * (x @ kappa) + phi)
    u = np.zeros(x.shape[:-1] + (d,))
    for a in range(d):
        for _ in range(modes):
            kappa = rng.integers(1, 4, size=d)
            phi = rng.uniform(0.0, 2.0 * np.pi)
            u[..., a] += u_amp * np.sin(2.0 * np.pi * (x @ kappa) + phi)
    return conserved(rho, u, np.ones_like(rho))


def smooth_density_wave(d, L, p):
    """Reference test state (``tests/conftest.py:30-39``): rho = 1 + 0.2
    sin(2 pi sum x), j_a = 0.5 rho, E = 1/0.4 + 0.5 rho d 0.25."""
    x = node_coordinates(d, L, p)
    rho = 1.0 + 0.2 * np.sin(2.0 * np.pi * np.sum(x, axis=-1))
    Q = np.zeros(x.shape[:-1] + (d + 2,))
    Q[..., 0] = rho
    for a in range(d):
        Q[..., 1 + a] = 0.5 * rho
    Q[..., -1] = 1.0 / 0.4 + 0.5 * rho * d * 0.25
    return Q


def uniform_state(d, L, p, state=None):
    """Constant state (``tests/test_scheduler.py:63-76``)."""
    n = p + 1
    if state is None:
        state = np.array([1.0] + [0.3, -0.1, 0.2][:d] + [2.5])
    return np.broadcast_to(np.asarray(state, dtype=float),
                           (3 ** (d * L),) + (n,) * d + (d + 2,)).copy()


GAUSSIAN_SIGMA = 0.25          # src/cli.py:30
ADVECTION_VELOCITY = (1.0, 0.5, 0.25)   # src/cli.py:31


def gaussian_profile(x):
    """Smooth periodic bump on the unit cube (src/cli.py:96-100)."""
    return np.exp(-np.sum(np.sin(np.pi * (x - 0.5)) ** 2, axis=-1)
                  / (2.0 * GAUSSIAN_SIGMA ** 2))


def gaussian_advect(d, L, p, noise=0.0, seed=0):
    """Scenario ``gaussian-advect`` (src/cli.py:139-142): q = gaussian_profile(x),
    m = 1; optional seeded U(-noise, noise) per node for harder parity cases."""
    x = node_coordinates(d, L, p)
    q = gaussian_profile(x)
    if noise:
        q = q + np.random.default_rng(seed).uniform(-noise, noise, size=q.shape)
    return q[..., None]


def shock_tube(d, L, p, seed=0, noise=0.0, pressure_ratio=10.0):
    """Periodic two-shock tube along x_0 (the reference's Sod states,
    ``src/cli.py`` "sod" / ``tests/test_limiter.py:104-109``, made periodic):
    rho = 1, p = 1 for |x_0 - 0.5| < 0.25, else rho = 0.125, p = 1/ratio;
    at rest, optional seeded U(-noise, noise) on the density.  Drives the
    subcell limiter (troubled cells at both discontinuities)."""
    x = node_coordinates(d, L, p)
    inside = np.abs(x[..., 0] - 0.5) < 0.25
    rho = np.where(inside, 1.0, 0.125)
    if noise:
        rho = rho + np.random.default_rng(seed).uniform(-noise, noise, size=rho.shape)
    pr = np.where(inside, 1.0, 1.0 / pressure_ratio)
    return conserved(rho, np.zeros(x.shape[:-1] + (d,)), pr)


def sod(d, L, p):
    """The reference's Sod tube (``src/cli.py:145-155``, ``tests/test_limiter.py:104-109``):
    rho = 1 / 0.125 and E = 1/0.4 / 0.1/0.4 left / right of x_0 = 0.5, at rest;
    run with outflow boundaries."""
    x = node_coordinates(d, L, p)
    left = x[..., 0] < 0.5
    Q = np.zeros(x.shape[:-1] + (d + 2,))
    Q[..., 0] = np.where(left, 1.0, 0.125)
    Q[..., -1] = np.where(left, 1.0, 0.1) / 0.4
    return Q


#: scenarios whose grid has outflow boundaries (src/cli.py:155)
OUTFLOW = ("sod",)

SCENARIOS = {
    "sod": sod,
    "shocktube": shock_tube,
    "bump": gaussian_bump_noise,
    "fourier": random_fourier,
    "wave": smooth_density_wave,
    "uniform": uniform_state,
    "gauss": gaussian_advect,
}


def build(name, d, L, p, **kw):
    if name not in SCENARIOS:
        raise ValueError(f"unknown scenario {name!r}; choose from {sorted(SCENARIOS)}")
    return np.ascontiguousarray(SCENARIOS[name](d, L, p, **kw), dtype=np.float64)
