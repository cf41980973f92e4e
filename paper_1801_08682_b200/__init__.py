"""B200-native (sm_100a) fused ADER-DG step for compressible Euler on periodic
Cartesian grids — drop-in for the reference's fused driver seam
(``/root/reference/pkg/src/aderdg/scheduler.py`` ``Driver(..., "fused")``).

Host code is Python; every realisation step runs as hand-written CUDA kernels
behind the C ABI declared in ``include/aderdg_b200.h``.  There is no CPU
fallback: importing works without a GPU, but constructing a ``Driver`` needs
the in-tree ``libaderdg_b200.so`` and a CUDA device.
"""

from .basis import Basis1D, make_basis
from .errors import (ConfigurationError, DeviceError, DomainError, NumericalError,
                     PredictorFailureError, ResourceBudgetError, SchedulingOrderError)
from .solver import (AdvectionSystem, Driver, EulerSystem, Grid, Kernels, TimeControl, build_grid,
                     device_bytes, gather, traversal_order)
from .limiter import SubcellLimiter, subcell_average_matrix

__version__ = "0.1.0"

__all__ = [
    "Basis1D", "ConfigurationError", "DeviceError", "DomainError", "Driver",
    "AdvectionSystem", "EulerSystem", "Grid", "Kernels", "NumericalError", "PredictorFailureError",
    "ResourceBudgetError", "SchedulingOrderError", "TimeControl", "build_grid",
    "device_bytes", "gather", "make_basis", "SubcellLimiter", "subcell_average_matrix",
    "traversal_order",
]
