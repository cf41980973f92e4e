"""A-posteriori subcell finite-volume limiter (reference ``src/limiter.py:26-234``).

``SubcellLimiter(system, basis, grid, cfl=0.9)`` is the configuration object the
reference hands to ``Driver(..., "straightforward", limiter=lim)``
(``src/scheduler.py:92-102``).  Here it carries the host-side setup operators —
the subcell-average matrix ``P``, its least-squares lift ``R``, the
nearest-node and node-to-subcell index maps — which ``Driver`` uploads with
``adg_set_limiter``; detection, the FV sub-steps and the reconstruction run
as sm_100a kernels (``csrc/aderdg_limiter.cuh``) after every corrector pass.
There is no host evaluation path for the limiter itself.
"""

import numpy as np

from .basis import subcell_operators
from .errors import ConfigurationError

DMP_ABS = 1e-3      # src/limiter.py:23 (compiled into lim_detect_kernel)
DMP_REL = 1e-2      # src/limiter.py:24


def subcell_average_matrix(basis):
    """src/limiter.py:26-34: ``P[s, i]`` = average of Lagrange polynomial i over
    subcell s of the unit interval split into 2p+1 equal parts (tabulated)."""
    return subcell_operators(basis.p)[0]


class SubcellLimiter:
    """src/limiter.py:87-108 (operators only; the limiting pass is on the GPU)."""

    def __init__(self, system, basis, grid, cfl=0.9):
        if getattr(system, "name", None) not in ("euler", "advection"):
            raise ConfigurationError("the GPU limiter is instantiated for the Euler and advection systems only")
        self.system = system
        self.basis = basis
        self.grid = grid
        self.cfl = cfl
        self.ns = 2 * basis.p + 1
        self.h_sub = grid.h / self.ns
        self.P, self.R = subcell_operators(basis.p)                # src/limiter.py:26-34,99
        w = basis.weights
        W = np.ones((basis.n,) * grid.d)
        for a in range(grid.d):
            W = W * w.reshape([basis.n if b == a else 1 for b in range(grid.d)])
        self.mean_weights = W[..., None]
        centers = (np.arange(self.ns) + 0.5) / self.ns
        self._nearest_node = np.argmin(np.abs(centers[:, None] - basis.nodes[None, :]), axis=1)
        # node -> subcell of the piecewise-constant fallback (src/limiter.py:227-228)
        self._node_subcell = np.minimum((basis.nodes * self.ns).astype(int), self.ns - 1)

    def device_arrays(self):
        """Contiguous arrays in the layout ``adg_set_limiter`` expects."""
        return (np.ascontiguousarray(self.P, dtype=np.float64),
                np.ascontiguousarray(self.R, dtype=np.float64),
                np.ascontiguousarray(self._nearest_node, dtype=np.int32),
                np.ascontiguousarray(self._node_subcell, dtype=np.int32))
