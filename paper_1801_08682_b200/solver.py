"""Drop-in host surface of the fused ADER-DG driver (reference driver seam).

Mirrors the reference's library use (``pkg/README.md:85-98``,
``tests/conftest.py:42-79``)::

    basis = make_basis(p)
    grid = build_grid(d, L, p, system.m)
    init: grid.cells[i].Q[...] = ...          (or grid.Q[...] = array)
    kernels = Kernels(EulerSystem(d), basis, grid, None, cfl=0.9)
    driver = Driver(grid, kernels, TimeControl(c_dt=0.99), "fused")
    driver.run(steps=N)
    Q = gather(grid); driver.step_records

Every realisation step runs on the GPU through the C ABI
(``include/aderdg_b200.h``): one call per step (``adg_step``) or per run
(``adg_run``).  The per-cell task methods of the reference ``Kernels`` class are
not re-exposed: the GPU replaces the whole driver seam, and
the PDE callbacks are compiled into the kernels (Euler, d = 2, 3).

Reference citations (``src/`` = ``/root/reference/pkg/src/aderdg/``):
  build_grid / Grid / Cell   src/mesh.py:27-243
  EulerSystem                src/pde.py:16-67
  Kernels (config)           src/kernels.py:37-60
  TimeControl                src/scheduler.py:35-74
  Driver (fused)             src/scheduler.py:88-226, 370-481
"""

import ctypes
import math
import time
from collections import Counter

import numpy as np

from . import _lib
from .basis import make_basis
from .errors import ConfigurationError, ResourceBudgetError

DEFAULT_CFL = 0.9                 # src/kernels.py:21
DEFAULT_C_DT = 0.99               # src/scheduler.py:32
DEFAULT_BUDGET_BYTES = None       # the reference's 2 GiB guard targets host RAM; HBM is 180 GB
GAMMA = 1.4


class EulerSystem:
    """Compressible Euler in d = 2, 3 (src/pde.py:16-67).  The flux,
    signal-speed and admissibility callbacks are compiled into the sm_100a
    kernels; this object selects the instantiation and offers the same
    pointwise functions on host arrays for setup and checks."""

    def __init__(self, dim):
        if dim not in (2, 3):
            from .errors import DomainError
            raise DomainError(f"Euler system supports d in {{2, 3}}, got {dim}")
        self.d = dim
        self.m = dim + 2
        self.name = "euler"

    def pressure(self, Q):
        Q = np.asarray(Q, dtype=float)
        j = Q[..., 1:1 + self.d]
        return (GAMMA - 1.0) * (Q[..., -1] - 0.5 * np.sum(j * j, axis=-1) / Q[..., 0])

    def max_signal_speed(self, Q, axis):
        Q = np.asarray(Q, dtype=float)
        rho = Q[..., 0]
        return np.abs(Q[..., 1 + axis] / rho) + np.sqrt(GAMMA * self.pressure(Q) / rho)

    def is_admissible(self, Q):
        Q = np.asarray(Q, dtype=float)
        if not np.all(np.isfinite(Q)):
            return False
        if not np.all(Q[..., 0] > 1e-12):
            return False
        return bool(np.all(self.pressure(Q) > 1e-12))


class AdvectionSystem:
    """Scalar linear advection ``q_t + v . grad q = 0`` (src/pde.py:70-102).
    The flux ``v_a q``, the signal speed ``|v_a|`` and the finiteness test are
    compiled into the generic sm_100a sweep kernel (``AdvectionPDE``); the
    velocity travels in ``adg_config.velocity``.  ``exact_solution`` is the
    analytic oracle of the convergence study (host-side post-processing)."""

    def __init__(self, dim, velocity, profile=None):
        from .errors import DomainError
        self.d = dim
        self.m = 1
        self.name = "advection"
        self.velocity = np.asarray(velocity, dtype=float)
        if self.velocity.shape != (dim,):
            raise DomainError(f"velocity must have {dim} components")
        self.profile = profile

    def max_signal_speed(self, Q, axis):
        Q = np.asarray(Q, dtype=float)
        return np.full(Q.shape[:-1], abs(self.velocity[axis]))

    def is_admissible(self, Q):
        return bool(np.all(np.isfinite(np.asarray(Q, dtype=float))))

    def exact_solution(self, x, t):
        from .errors import DomainError
        if self.profile is None:
            raise DomainError("advection system has no initial profile attached")
        shifted = np.mod(np.asarray(x, dtype=float) - t * self.velocity, 1.0)
        return self.profile(shifted)[..., None]


class Cell:
    """Reference Cell view (src/mesh.py:27-40): ``Q`` is a view into the
    grid's contiguous state array."""

    __slots__ = ("index", "multi_index", "Q")

    def __init__(self, index, multi_index, Q):
        self.index = index
        self.multi_index = multi_index
        self.Q = Q


class _CellList:
    """Lazily materialised ``grid.cells`` (531441 cells at 81^3)."""

    def __init__(self, grid):
        self._g = grid

    def __len__(self):
        return self._g.n_cells

    def __getitem__(self, i):
        g = self._g
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        i = int(i)
        if i < 0:
            i += g.n_cells
        if not 0 <= i < g.n_cells:
            raise IndexError(i)
        multi = tuple(int(v) for v in np.unravel_index(i, (g.cells_per_axis,) * g.d))
        return Cell(i, multi, g.Q[i])

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]


class Grid:
    """Periodic 3^L-per-axis Cartesian grid on the unit cube (src/mesh.py:63-146).

    ``Q`` holds every cell's coefficients in reference order
    ``(n_cells,) + (p+1,)*d + (m,)``; ``cells[i].Q`` views into it."""

    def __init__(self, d, L, p, m, boundary="periodic", storage="hull"):
        self.d, self.L, self.p, self.m = d, L, p, m
        self.boundary = boundary
        self.storage = storage
        self.h = 3.0 ** (-L)                       # src/mesh.py:71
        n = p + 1
        self.Q = np.zeros((3 ** (d * L),) + (n,) * d + (m,))
        self.cells = _CellList(self)

    @property
    def n_cells(self):
        return 3 ** (self.d * self.L)

    @property
    def cells_per_axis(self):
        return 3 ** self.L

    def node_block_shape(self):
        return (self.p + 1,) * self.d + (self.m,)

    def persistent_doubles(self, include_limiter=False):
        """src/mesh.py:124-137: doubles the reference allocates for this grid
        (its storage layout; the GPU's own HBM is ``device_bytes``)."""
        from .metrics import estimate_persistent_doubles
        return estimate_persistent_doubles(self.d, self.L, self.p, self.m, self.boundary, self.storage)


def device_bytes(d, L, p, m=None):
    """Persistent HBM of one single-GPU solver: Q, D and two parities of
    time-collapsed face records (2d per cell, 2 n^(d-1) m + 2 doubles each)."""
    n, cells = p + 1, 3 ** (d * L)
    m = d + 2 if m is None else m
    rec = 2 * n ** (d - 1) * m + 2
    slots = (3 ** L + 2) * 3 ** (L * (d - 1))
    return 8 * (2 * cells * n ** d * m + 2 * 2 * d * slots * rec)


def build_grid(d, L, p, m, boundary="periodic", storage="hull",
               budget_bytes=DEFAULT_BUDGET_BYTES):
    """src/mesh.py:167-243 (periodic or outflow boundaries; the device layout
    is the same for both storage kinds)."""
    if d not in (2, 3):
        raise ConfigurationError(f"dimension must be 2 or 3, got {d}")
    if not 1 <= L <= 4:
        raise ConfigurationError(f"depth L must be in [1, 4], got {L}")
    if not 0 <= p <= 9:
        raise ConfigurationError(f"order p must be in [0, 9], got {p}")
    if boundary not in ("periodic", "outflow"):
        raise ConfigurationError(f"unknown boundary kind {boundary!r}")
    if storage not in ("hull", "spacetime"):
        raise ConfigurationError(f"unknown storage layout {storage!r}")
    if m not in (d + 2, 1):
        raise ConfigurationError(f"the GPU path implements Euler (m = d+2) and advection (m = 1), got m={m}")
    if budget_bytes is not None:
        req = device_bytes(d, L, p, m)
        if req > budget_bytes:
            raise ResourceBudgetError(req, budget_bytes)
    return Grid(d, L, p, m, boundary, storage)


class Kernels:
    """Configuration carrier of the reference kernel suite (src/kernels.py:46-60)."""

    def __init__(self, system, basis, grid, ledger=None, cfl=DEFAULT_CFL):
        if getattr(system, "name", None) not in ("euler", "advection"):
            raise ConfigurationError("the GPU kernels are instantiated for the Euler and advection systems only")
        if system.d != grid.d or basis.p != grid.p or system.m != grid.m:
            raise ConfigurationError("system / basis / grid disagree on d or p")
        self.system, self.basis, self.grid = system, basis, grid
        self.ledger = ledger
        self.cfl = cfl
        w = basis.weights
        self.kvol = (basis.diff.T * w[None, :]) / w[:, None]
        self.lift_low = basis.left / w
        self.lift_high = basis.right / w
        self.picard_cap = max(1, 2 * basis.n)


class TimeControl:
    """src/scheduler.py:35-74; mirrors the device time control after each sync."""

    def __init__(self, c_dt=DEFAULT_C_DT, averaging="strict", forced_dt=None):
        if not 0.0 < c_dt <= 1.0:
            raise ConfigurationError(f"c_dt must be in (0, 1], got {c_dt}")
        if averaging not in ("strict", "creeping"):
            raise ConfigurationError(f"unknown averaging mode {averaging!r}")
        self.c_dt, self.averaging, self.forced_dt = c_dt, averaging, forced_dt
        self.T, self.dt_old, self.dt_new, self.dt_adm = 0.0, 0.0, 0.0, math.inf


def _config(grid, kernels, tc, inject_rerun, spike_step, spike_factor, device, rank=0, world=1,
            mode="fused"):
    cfg = _lib.AdgConfig()
    cfg.d, cfg.p, cfg.L = grid.d, grid.p, grid.L
    cfg.cfl = float(kernels.cfl)
    cfg.c_dt = float(tc.c_dt)
    cfg.creeping = 1 if tc.averaging == "creeping" else 0
    cfg.forced_dt = float("nan") if tc.forced_dt is None else float(tc.forced_dt)
    cfg.inject_rerun = 1 if inject_rerun else 0
    cfg.spike_step = -1 if spike_step is None else int(spike_step)
    cfg.spike_factor = float(spike_factor)
    cfg.device = int(device)
    cfg.rank, cfg.world = int(rank), int(world)
    cfg.driver_mode = 1 if mode == "straightforward" else 0
    cfg.boundary = 1 if grid.boundary == "outflow" else 0
    system = kernels.system
    if system.name == "advection":
        cfg.system = 1
        for a in range(grid.d):
            cfg.velocity[a] = float(system.velocity[a])
    return cfg


def upload_operators(handle, basis):
    ops = [np.ascontiguousarray(a, dtype=np.float64) for a in
           (basis.nodes, basis.weights, basis.diff, basis.integ, basis.left, basis.right)]
    handle.call("adg_set_operators", *[_lib.dptr(a) for a in ops])
    return ops


def _peano_order(d, L):
    """Cells along the d-dimensional Peano curve of depth L (src/mesh.py:246-275):
    base-3 digits of the curve parameter go round-robin to the axes, coarsest
    first; a digit is mirrored when the digits seen so far on the other axes
    sum to an odd number."""
    K = 3 ** L
    out = np.empty(K ** d, dtype=np.int64)
    for t in range(K ** d):
        digits = np.base_repr(t, 3).rjust(d * L, "0") if t else "0" * (d * L)
        coords = [0] * d
        others = [0] * d
        for i, ch in enumerate(digits):
            a, dig = i % d, int(ch)
            coords[a] = coords[a] * 3 + (2 - dig if others[a] % 2 else dig)
            for b in range(d):
                if b != a:
                    others[b] += dig
        out[t] = np.ravel_multi_index(coords, (K,) * d)
    return out


def traversal_order(grid, kind):
    """src/mesh.py:278-286: cell order of a sweep ("lexicographic" or "peano")."""
    if kind == "lexicographic":
        return np.arange(grid.n_cells, dtype=np.int64)
    if kind == "peano":
        return _peano_order(grid.d, grid.L)
    raise ConfigurationError(f"unknown traversal kind {kind!r}")


class Driver:
    """GPU driver (src/scheduler.py:88-313): the fused single-touch mode (the
    north-star path) or the straightforward three-sweep mode (predict pass,
    Riemann + corrector pass; dt = dt_new, no priming, no rerun).

    ``host_sync``: "step" copies the state back into ``grid.Q`` after every
    step (reference semantics: ``cell.Q`` is current after ``step()``);
    "run" only at the end of ``run()``; "manual" never (call ``sync_state``).
    """

    def __init__(self, grid, kernels, time_control, mode="fused",
                 traversal="lexicographic", parallel=False, n_workers=4,
                 inject_rerun=False, spike_step=None, spike_factor=3.0,
                 limiter=None, device=0, host_sync="step", devices=None, debug_checks=False):
        if mode not in ("straightforward", "shifted", "fused"):
            raise ConfigurationError(f"unknown scheduler mode {mode!r}")
        if mode == "shifted":
            raise ConfigurationError("the shifted driver is not implemented on the GPU (out of scope)")
        if parallel and mode == "shifted":
            raise ConfigurationError("the shifted driver is sequential only")
        if limiter is not None and mode != "straightforward":       # src/scheduler.py:100-102
            raise ConfigurationError("subcell limiting is supported in straightforward mode only")
        if isinstance(traversal, np.ndarray):
            if sorted(traversal.tolist()) != list(range(grid.n_cells)):
                raise ConfigurationError("traversal must be a permutation of the cells")
        elif traversal not in ("lexicographic", "peano"):
            raise ConfigurationError(f"unknown traversal kind {traversal!r}")
        if spike_step is not None and kernels.system.name != "euler":
            raise ConfigurationError("the speed spike is defined for Euler runs")
        if host_sync not in ("step", "run", "manual"):
            raise ConfigurationError(f"unknown host_sync {host_sync!r}")
        # the fused result is traversal-invariant (tests/test_scheduler.py:111-116):
        # all cells of a sweep run concurrently on the GPU.
        self.grid, self.kernels, self.tc, self.mode = grid, kernels, time_control, mode
        self.traversal, self.parallel, self.n_workers = traversal, parallel, n_workers
        self.inject_rerun, self.spike_step, self.spike_factor = inject_rerun, spike_step, spike_factor
        self.limiter = limiter
        self.order = traversal if isinstance(traversal, np.ndarray) else traversal_order(grid, traversal)
        self.host_sync = host_sync
        self.sweep_count = self.step_count = self.rerun_count = 0
        self.reruns_by_step = Counter()
        self.troubled_by_step = Counter()
        self.step_records = []
        self.picard_iters = 0
        self.predicts = 0
        self.devices = self._slab_devices(parallel, n_workers, device, devices)
        self.group = None
        if len(self.devices) > 1:
            from .parallel import SlabGroup
            self.group = SlabGroup(
                lambda: _config(grid, kernels, time_control, inject_rerun, spike_step, spike_factor,
                                device, mode=mode),
                self.devices, kernels.basis, grid.d, grid.p)
            self.handle = self.group.lead
            self.group.load(grid.Q)
            self.group.seed()                             # Driver._seed_time_control (global)
            self._pull_tc()
            return
        cfg = _config(grid, kernels, time_control, inject_rerun, spike_step, spike_factor, device,
                      mode=mode)
        # debug_checks: the ADG_DEBUG_CHECKS build of the same kernels (stale-record and
        # bounds checks, poisoned shared memory, jittered barriers; DeviceError on a hit)
        self.handle = _lib.Handle(cfg, debug=debug_checks)
        self._ops = upload_operators(self.handle, kernels.basis)
        if limiter is not None:
            # SubcellLimiter operators + the traversal that fixes whose prev_Q the
            # DMP test sees (src/limiter.py:138-160, src/kernels.py:208-214)
            P, R, nearest, sample = limiter.device_arrays()
            order = np.ascontiguousarray(self.order, dtype=np.int64)
            self._lim_arrays = (P, R, nearest, sample, order)
            self.handle.call("adg_set_limiter", _lib.dptr(P), _lib.dptr(R),
                             nearest.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                             sample.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                             order.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)),
                             ctypes.c_double(float(limiter.cfl)))
        self.load_state(grid.Q)
        self.handle.call("adg_seed")                       # Driver._seed_time_control
        self._pull_tc()

    def _slab_devices(self, parallel, n_workers, device, devices):
        """GPUs of the run.  The reference's ``parallel=True, n_workers=N`` runs the
        per-cell tasks on a thread pool (src/scheduler.py:126-130); on the GPU every
        cell of a sweep already runs concurrently, so the workers become x-slabs of the
        grid on N GPUs of this process (at most the visible GPUs and the 3^L cell planes).
        ``devices`` names them explicitly.  Limited or outflow runs stay on one GPU
        (those paths run on a single slab)."""
        if devices is not None:
            devs = [int(x) for x in devices]
            if len(set(devs)) != len(devs) or not devs:
                raise ConfigurationError("devices must be distinct GPU ordinals")
        elif parallel:
            visible = _lib.load_library().adg_device_count()
            want = max(1, int(n_workers))
            devs = [(device + i) % max(visible, 1) for i in range(min(want, max(visible, 1)))]
        else:
            return [int(device)]
        if len(devs) > 1:
            if self.limiter is not None or self.grid.boundary != "periodic":
                return [devs[0]]
            devs = devs[:self.grid.cells_per_axis]
        return devs

    # -- state transfer ------------------------------------------------------
    def load_state(self, Q):
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        if self.group is not None:
            self.group.load(Q)
            return
        self.handle.call("adg_load_state", _lib.dptr(Q), Q.size)

    def sync_state(self):
        """Copy the device state into ``grid.Q`` (``grid.cells[i].Q``)."""
        Q = self.grid.Q
        if not Q.flags.c_contiguous:
            raise ConfigurationError("grid.Q must stay C-contiguous")
        if self.group is not None:
            self.group.store(Q)
            return Q
        self.handle.call("adg_store_state", _lib.dptr(Q), Q.size)
        return Q

    def _pull_tc(self):
        T, dt_old, dt_new, dt_adm = self.handle.time_control()
        self.tc.T, self.tc.dt_old, self.tc.dt_new, self.tc.dt_adm = T, dt_old, dt_new, dt_adm

    def _book_ledger(self, r, rec):
        """Access counts of step ``r.step`` in the reference's ledger units
        (src/scheduler.py:459-481 with src/metrics.py:157-175); see metrics.py."""
        from . import metrics
        led = self.kernels.ledger
        if led is None or not hasattr(led, "book"):
            return
        g = self.grid
        K = g.cells_per_axis
        n_faces = g.d * g.n_cells if g.boundary == "periodic" else g.d * (K + 1) * K ** (g.d - 1)
        rec.update(metrics.record_step(led, self.mode, r.step, r.reruns, g.n_cells, n_faces,
                                       int(r.troubled)))

    def _absorb(self, recs, wall_time=0.0):
        for r in recs:
            if r.reruns:
                self.reruns_by_step[r.step] += r.reruns
            if r.troubled:
                self.troubled_by_step[r.step] = int(r.troubled)
            self.picard_iters += r.picard_iters
            self.predicts += r.predicts
            rec = {
                "step": r.step, "T": r.T, "dt_old": r.dt_old, "dt_new": r.dt_new,
                "dt_adm": r.dt_adm, "reruns": r.reruns, "troubled": int(r.troubled),
                "wall_time": wall_time / max(1, len(recs)),
                "picard_iters": r.picard_iters, "predicts": r.predicts,
            }
            self._book_ledger(r, rec)
            self.step_records.append(rec)
        lib, h = self.handle.lib, self.handle.h
        self.step_count = lib.adg_step_count(h)
        self.rerun_count = lib.adg_rerun_count(h)
        self.sweep_count = lib.adg_sweep_count(h)
        self._pull_tc()

    def _finish(self, recs, err, wall_time=0.0):
        self._absorb(recs, wall_time)
        if err is not None:
            raise err

    # -- public API (src/scheduler.py:190-226) --------------------------------
    def step(self):
        rec = _lib.AdgStepRecord()
        t0 = time.perf_counter()
        if self.group is not None:
            st = self.group.run(1, (_lib.AdgStepRecord * 1).from_address(ctypes.addressof(rec)))
        else:
            st = self.handle.lib.adg_step(self.handle.h, rec)
        wall = time.perf_counter() - t0
        err = None
        try:
            self.handle.check(st, "adg_step")
        except Exception as e:  # keep the driver's counters consistent before raising
            err = e
        self._finish([rec] if st == 0 else [], err, wall)
        if self.host_sync == "step":
            self.sync_state()
        return self.step_count

    def run(self, steps=None, final_time=None):
        if (steps is None) == (final_time is None):
            raise ConfigurationError("specify exactly one of steps / final_time")
        if final_time is not None:
            if self.mode != "straightforward":
                raise ConfigurationError(
                    "final-time integration requires the straightforward driver "
                    "(the pipelined modes realise steps one sweep late)")
            return self._run_to(float(final_time))
        steps = int(steps)
        if steps <= 0:
            return self.step_count
        recs = (_lib.AdgStepRecord * steps)()
        before = self.step_count
        t0 = time.perf_counter()
        if self.group is not None:
            st = self.group.run(steps, recs)
        else:
            st = self.handle.lib.adg_run(self.handle.h, steps, recs)
        wall = time.perf_counter() - t0
        err = None
        try:
            self.handle.check(st, "adg_run")
        except Exception as e:
            err = e
        done = self.handle.lib.adg_step_count(self.handle.h) - before
        if self.host_sync in ("step", "run"):
            self.sync_state()
        self._finish(list(recs)[:done], err, wall)
        return self.step_count

    def _run_to(self, final_time):
        """src/scheduler.py:223-226: clamp dt_new so the last step lands on final_time."""
        while True:
            T, dt_old, dt_new, dt_adm = self.handle.time_control()
            if not T < final_time - 1e-14:
                break
            if dt_new > final_time - T:
                for h in (self.group.handles if self.group is not None else [self.handle]):
                    h.call("adg_set_dt_new", ctypes.c_double(final_time - T))
            self.step()
        return self.step_count

    def troubled_flags(self):
        """``[cell.troubled for cell in grid.cells]`` (src/mesh.py:39): set by the
        limiter pipeline, cleared by a successful reconstruction."""
        out = np.zeros(self.grid.n_cells, dtype=np.uint8)
        self.handle.call("adg_troubled_flags", out.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte)),
                         out.size)
        return out.astype(bool)

    def picard_histogram(self):
        """Picard iterations per predict, summed over every predict so far."""
        h = self.group.picard_histogram() if self.group is not None else self.handle.picard_histogram()
        return {int(k): int(v) for k, v in enumerate(h) if v}

    def close(self):
        if self.group is not None:
            self.group.close()
        else:
            self.handle.close()


def gather(grid):
    """tests/conftest.py:77-79."""
    return np.array(grid.Q)


__all__ = ["EulerSystem", "AdvectionSystem", "Grid", "Cell", "build_grid", "Kernels", "TimeControl",
           "Driver", "gather", "make_basis", "device_bytes"]
