"""CPU oracle for the fused ADER-DG Euler step — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The product path (``paper_1801_08682_b200``)
never imports anything under ``oracle/`` and fails loudly when its CUDA
library is missing.

What it is: a batched numpy restatement of the reference's fused
(single-touch, optimistic) driver for the compressible Euler equations on a
periodic Cartesian grid.  Where the reference loops over cells in Python and
calls numpy per cell, this file runs every task on all cells at once, so the
arithmetic per cell is the reference's arithmetic (same operators, same
formulas, same task order) while the batching only changes BLAS summation
order inside the small tensordots.

Pinning: ``tests/test_oracle_golden.py`` checks this oracle against golden
vectors produced by the reference itself (``tests/golden/make_golden.py``
imports ``/root/reference/pkg/src/aderdg`` in the build container and writes
``tests/golden/*.npz``).  Observed agreement: <=1e-13 relative L-inf.

Reference citations (``src/`` = ``/root/reference/pkg/src/aderdg/``):
  basis       src/basis.py:31-122         make_basis / Gauss-Legendre / lagrange_eval
  pde         src/pde.py:12-67            EulerSystem pressure / flux / speed / admissible
              src/pde.py:70-94            AdvectionSystem flux / speed / admissible
  kernels     src/kernels.py:46-229       predict / extrapolate / integrate_volume /
                                          solve_riemann / integrate_face / update /
                                          calc_time_step
  time ctl    src/scheduler.py:35-85      TimeControl / update_time_step_sizes
  driver      src/scheduler.py:135-155    _seed_time_control
              src/scheduler.py:190-208    step (priming sweep on first call)
              src/scheduler.py:370-449    _maybe_rerun / _sweep_fused
              src/scheduler.py:459-481    _record_step
  topology    src/mesh.py:167-243         periodic faces, cell_faces order
"""

from collections import Counter

import numpy as np

GAMMA = 1.4                 # src/pde.py:12
ADMISSIBILITY_EPS = 1e-12   # src/pde.py:13
DEFAULT_CFL = 0.9           # src/kernels.py:21
DEFAULT_C_DT = 0.99         # src/scheduler.py:32
MAX_ORDER = 9               # src/basis.py:13
_NEWTON_TOL = 1e-15         # src/basis.py:15


class OracleError(RuntimeError):
    """Raised by the oracle with the reference's error class name and the
    failing cell (first in lexicographic traversal order)."""

    def __init__(self, kind, message, cell_index=None, step=None):
        self.kind = kind              # "NumericalError" | "PredictorFailureError"
        self.cell_index = cell_index
        self.step = step
        super().__init__(f"{kind}: {message}")


# ---------------------------------------------------------------------------
# basis (src/basis.py:18-122)

def _legendre_and_derivative(n, x):
    """src/basis.py:18-28."""
    p_prev = np.ones_like(x)
    p = x.copy()
    if n == 0:
        return p_prev, np.zeros_like(x)
    for k in range(2, n + 1):
        p_prev, p = p, ((2 * k - 1) * x * p - (k - 1) * p_prev) / k
    dp = n * (x * p - p_prev) / (x * x - 1.0)
    return p, dp


def _gauss_legendre_unit(n):
    """src/basis.py:31-52: Newton on the Legendre recurrence, mapped to (0,1)."""
    if n == 1:
        return np.array([0.5]), np.array([1.0])
    k = np.arange(1, n + 1)
    x = np.cos(np.pi * (k - 0.25) / (n + 0.5))
    for _ in range(100):
        p, dp = _legendre_and_derivative(n, x)
        dx = p / dp
        x = x - dx
        if np.max(np.abs(dx)) < _NEWTON_TOL:
            break
    p, dp = _legendre_and_derivative(n, x)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    order = np.argsort(x)
    x, w = x[order], w[order]
    return 0.5 * (x + 1.0), 0.5 * w


def lagrange_eval(nodes, points):
    """src/basis.py:55-66."""
    nodes = np.asarray(nodes, dtype=float)
    points = np.atleast_1d(np.asarray(points, dtype=float))
    n = nodes.size
    L = np.ones((points.size, n))
    for j in range(n):
        for k in range(n):
            if k == j:
                continue
            L[:, j] *= (points - nodes[k]) / (nodes[j] - nodes[k])
    return L


class Basis:
    __slots__ = ("p", "n", "nodes", "weights", "diff", "left", "right", "integ")


def make_basis(p):
    """src/basis.py:91-122."""
    if not isinstance(p, (int, np.integer)) or not 0 <= p <= MAX_ORDER:
        raise ValueError(f"order p must be an integer in [0, {MAX_ORDER}], got {p!r}")
    n = p + 1
    nodes, weights = _gauss_legendre_unit(n)
    bary = np.ones(n)
    for j in range(n):
        for k in range(n):
            if k != j:
                bary[j] /= nodes[j] - nodes[k]
    diff = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if i != j:
                diff[i, j] = (bary[j] / bary[i]) / (nodes[i] - nodes[j])
        diff[i, i] = -np.sum(diff[i, :])
    left = lagrange_eval(nodes, 0.0)[0]
    right = lagrange_eval(nodes, 1.0)[0]
    integ = np.zeros((n, n))
    for i in range(n):
        sub = nodes * nodes[i]
        integ[i, :] = nodes[i] * (weights @ lagrange_eval(nodes, sub))
    b = Basis()
    b.p, b.n, b.nodes, b.weights, b.diff = p, n, nodes, weights, diff
    b.left, b.right, b.integ = left, right, integ
    return b


def apply_matrix(mat, arr, axis):
    """src/basis.py:148-150 (``axis`` counts the leading cell axis here)."""
    return np.moveaxis(np.tensordot(mat, arr, axes=(1, axis)), 0, axis)


# ---------------------------------------------------------------------------
# Euler system (src/pde.py:16-67); arrays carry a leading cell axis

def pressure(Q, d):
    """src/pde.py:27-32."""
    rho = Q[..., 0]
    j = Q[..., 1:1 + d]
    E = Q[..., -1]
    return (GAMMA - 1.0) * (E - 0.5 * np.sum(j * j, axis=-1) / rho)


def flux(Q, d):
    """src/pde.py:34-49: flux tensor with shape (d,) + Q.shape."""
    rho = Q[..., 0]
    j = Q[..., 1:1 + d]
    E = Q[..., -1]
    p = pressure(Q, d)
    F = np.empty((d,) + Q.shape)
    for a in range(d):
        ja = j[..., a]
        F[a, ..., 0] = ja
        for b in range(d):
            F[a, ..., 1 + b] = ja * j[..., b] / rho
        F[a, ..., 1 + a] += p
        F[a, ..., -1] = ja * (E + p) / rho
    return F


def max_signal_speed(Q, axis, d):
    """src/pde.py:51-57."""
    rho = Q[..., 0]
    u = Q[..., 1 + axis] / rho
    c = np.sqrt(GAMMA * pressure(Q, d) / rho)
    return np.abs(u) + c


def admissible_per_cell(Q, d):
    """src/pde.py:59-67, one verdict per leading cell."""
    C = Q.shape[0]
    flat = Q.reshape(C, -1, Q.shape[-1])
    finite = np.all(np.isfinite(flat), axis=(1, 2))
    with np.errstate(all="ignore"):
        rho_ok = np.all(flat[..., 0] > ADMISSIBILITY_EPS, axis=1)
        p_ok = np.all(pressure(flat, d) > ADMISSIBILITY_EPS, axis=1)
    return finite & rho_ok & p_ok


class EulerPDE:
    """src/pde.py:16-67 as a plug-in of the batched kernels."""

    name = "euler"

    def __init__(self, d):
        self.d, self.m = d, d + 2

    def flux(self, Q):
        return flux(Q, self.d)

    def max_signal_speed(self, Q, axis):
        return max_signal_speed(Q, axis, self.d)

    def admissible_per_cell(self, Q):
        return admissible_per_cell(Q, self.d)


class AdvectionPDE:
    """src/pde.py:70-94: F_a = v_a q, speed |v_a|, admissible iff finite."""

    name = "advection"

    def __init__(self, d, velocity):
        self.d, self.m = d, 1
        self.velocity = np.asarray(velocity, dtype=float)[:d]

    def flux(self, Q):
        F = np.empty((self.d,) + Q.shape)
        for a in range(self.d):
            F[a] = self.velocity[a] * Q
        return F

    def max_signal_speed(self, Q, axis):
        return np.full(Q.shape[:-1], abs(self.velocity[axis]))

    def admissible_per_cell(self, Q):
        C = Q.shape[0]
        return np.all(np.isfinite(Q.reshape(C, -1)), axis=1)


# ---------------------------------------------------------------------------
# grid topology (src/mesh.py:167-243, periodic)

def neighbour_tables(d, K, outflow=False):
    """minus[a][c] / plus[a][c]: neighbour cell of c along axis a (src/mesh.py:202-231;
    cell index = C-order ravel, src/mesh.py:191-200); periodic wrap, or -1 across
    an outflow boundary."""
    shape = (K,) * d
    idx = np.arange(K ** d).reshape(shape)
    minus = [np.roll(idx, 1, axis=a).ravel() for a in range(d)]
    plus = [np.roll(idx, -1, axis=a).ravel() for a in range(d)]
    if outflow:
        for a in range(d):
            ia = np.unravel_index(np.arange(K ** d), shape)[a]
            minus[a] = np.where(ia == 0, -1, minus[a])
            plus[a] = np.where(ia == K - 1, -1, plus[a])
    return minus, plus


# ---------------------------------------------------------------------------
# the seven tasks, batched over cells

class OracleKernels:
    """Batched restatement of ``Kernels`` (src/kernels.py:37-229) for Euler."""

    def __init__(self, d, p, L, cfl=DEFAULT_CFL, pde=None, boundary="periodic"):
        self.d, self.p, self.L = d, p, L
        self.outflow = boundary == "outflow"
        self.pde = pde if pde is not None else EulerPDE(d)
        self.m = self.pde.m
        self.basis = b = make_basis(p)
        self.n = b.n
        self.K = 3 ** L
        self.h = 3.0 ** (-L)                      # src/mesh.py:71
        self.cfl = cfl
        w = b.weights
        self.kvol = (b.diff.T * w[None, :]) / w[:, None]   # src/kernels.py:56
        self.lift_low = b.left / w                          # src/kernels.py:58
        self.lift_high = b.right / w                        # src/kernels.py:59
        self.picard_cap = max(1, 2 * b.n)                   # src/kernels.py:60
        self.minus, self.plus = neighbour_tables(d, self.K, self.outflow)
        self.picard_hist = Counter()

    # src/kernels.py:68-105
    def predict(self, Q, dt, cells=None):
        """Q: (C, n..., m).  Returns (q, f, fail_mask, iters)."""
        b, d = self.basis, self.d
        C = Q.shape[0]
        fail = ~np.all(np.isfinite(Q.reshape(C, -1)), axis=1)
        Qb = Q[..., None, :]
        q = np.repeat(Qb, b.n, axis=-2)
        with np.errstate(all="ignore"):
            tol = 1e-10 * (1.0 + np.max(np.abs(Q.reshape(C, -1)), axis=1))
        scale = dt / self.h
        active = np.nonzero(~fail)[0]
        iters = np.zeros(C, dtype=np.int64)
        bshape = (-1,) + (1,) * (d + 2)
        for _ in range(self.picard_cap):
            if active.size == 0:
                break
            qa = q[active]
            with np.errstate(all="ignore"):
                F = self.pde.flux(qa)
                div = apply_matrix(b.diff, F[0], axis=1)
                for a in range(1, d):
                    div += apply_matrix(b.diff, F[a], axis=1 + a)
                sc = scale[active] if np.ndim(scale) else scale
                sc = np.reshape(sc, bshape) if np.ndim(sc) else sc
                q_new = Qb[active] - sc * apply_matrix(b.integ, div, axis=1 + d)
                delta = np.max(np.abs(q_new - qa).reshape(active.size, -1), axis=1)
            q[active] = q_new
            iters[active] += 1
            bad = ~np.isfinite(delta)
            fail[active[bad]] = True
            done = bad | (delta <= tol[active])
            active = active[~done]
        with np.errstate(all="ignore"):
            f = self.pde.flux(q)
        fail |= ~np.all(np.isfinite(f.reshape(d, C, -1)), axis=(0, 2))
        for k, v in Counter(iters[~fail].tolist()).items():
            self.picard_hist[k] += v
        return q, f, fail, iters

    # src/kernels.py:107-128: own-side traces for all 2d faces of each cell
    def extrapolate(self, q, f):
        """Returns tr_q[a][s], tr_f[a][s] with shape (C, n^(d-1) axes..., n, m):
        s = 0 low face (cell is its PLUS side), s = 1 high face (MINUS side)."""
        b, d = self.basis, self.d
        tr_q, tr_f = [], []
        for a in range(d):
            tq, tf = [], []
            for vec in (b.left, b.right):
                tq.append(np.tensordot(vec, q, axes=(0, 1 + a)))
                tf.append(np.tensordot(vec, f[a], axes=(0, 1 + a)))
            tr_q.append(tq)
            tr_f.append(tf)
        return tr_q, tr_f

    # src/kernels.py:130-143
    def integrate_volume(self, f, dt):
        b, d = self.basis, self.d
        fbar = np.tensordot(f, b.weights, axes=(d + 2, 0))  # (d, C, n..., m)
        D = apply_matrix(self.kvol, fbar[0], axis=1)
        for a in range(1, d):
            D += apply_matrix(self.kvol, fbar[a], axis=1 + a)
        D *= dt / self.h
        return D

    # src/kernels.py:147-179: one Rusanov solve per face (face = low face of cell c)
    def solve_riemann(self, tr_q, tr_f, populated=True):
        """Returns fstar[a] = (low, high) with shape (C, ...): F* of the low and
        the high face of each cell along axis a (low face: minus side = low
        neighbour's high trace).  At an outflow boundary face the ghost side
        holds the cell's own trace (src/kernels.py:124-127)."""
        d = self.d
        out = []
        for a in range(d):
            qp, fp = tr_q[a][0], tr_f[a][0]                 # plus side: own low trace
            qm = tr_q[a][1][self.minus[a]]                  # minus side: neighbour high
            fm = tr_f[a][1][self.minus[a]]
            if self.outflow:
                lo = (self.minus[a] < 0).reshape((-1,) + (1,) * (qp.ndim - 1))
                qm, fm = np.where(lo, qp, qm), np.where(lo, fp, fm)
            if not populated:
                out.append((np.zeros_like(qp), np.zeros_like(qp)))
                continue
            low = self._rusanov(qm, fm, qp, fp, a)
            high = low[self.plus[a]]
            if self.outflow:
                hi = (self.plus[a] < 0).reshape((-1,) + (1,) * (qp.ndim - 1))
                qh, fh = tr_q[a][1], tr_f[a][1]             # own high trace on both sides
                high = np.where(hi, self._rusanov(qh, fh, qh, fh, a), high)
            out.append((low, high))
        return out

    def _rusanov(self, qm, fm, qp, fp, a):
        """src/kernels.py:173-177 for one batch of faces."""
        C = qp.shape[0]
        with np.errstate(all="ignore"):
            sm = np.max(self.pde.max_signal_speed(qm, a).reshape(C, -1), axis=1)
            sp = np.max(self.pde.max_signal_speed(qp, a).reshape(C, -1), axis=1)
        # python max(sm, sp): a NaN on the minus side wins, one on the plus side is ignored
        alpha = np.where(np.isnan(sp), sm, np.maximum(sm, sp))
        al = alpha.reshape((-1,) + (1,) * (qp.ndim - 1))
        return 0.5 * (fm + fp) - 0.5 * al * (qp - qm)

    # src/kernels.py:183-206 (fixed order: axis ascending, low then high)
    def integrate_face(self, D, fstar, dt):
        b, d = self.basis, self.d
        scale = dt / self.h
        for a in range(d):
            for side_local, lift in ((0, self.lift_low), (1, self.lift_high)):
                if side_local == 0:
                    blk = -fstar[a][0]                    # PLUS side stores -F*
                else:
                    blk = fstar[a][1]                     # MINUS side stores +F*
                fbar = np.tensordot(blk, b.weights, axes=(d, 0))   # (C, n^(d-1)..., m)
                shape = [1] * (d + 2)
                shape[1 + a] = b.n
                D -= scale * lift.reshape(shape) * np.expand_dims(fbar, 1 + a)
        return D

    # src/kernels.py:216-229 -> per-cell admissible dt (None -> nan + flag)
    def calc_time_step(self, Q):
        d = self.d
        C = Q.shape[0]
        ok = self.pde.admissible_per_cell(Q)
        lam = np.zeros(C)
        with np.errstate(all="ignore"):
            for a in range(d):
                lam = np.maximum(lam, np.max(self.pde.max_signal_speed(Q, a).reshape(C, -1), axis=1))
            dt = self.cfl * self.h / (d * (2 * self.p + 1) * lam)
        dt = np.where(lam <= 0.0, np.inf, dt)
        return dt, ok, lam


# ---------------------------------------------------------------------------
# time control (src/scheduler.py:35-85)

class TimeControl:
    def __init__(self, c_dt=DEFAULT_C_DT, averaging="strict", forced_dt=None):
        if not 0.0 < c_dt <= 1.0:
            raise ValueError(f"c_dt must be in (0, 1], got {c_dt}")
        if averaging not in ("strict", "creeping"):
            raise ValueError(f"unknown averaging mode {averaging!r}")
        self.c_dt, self.averaging, self.forced_dt = c_dt, averaging, forced_dt
        self.T, self.dt_old, self.dt_new, self.dt_adm = 0.0, 0.0, 0.0, np.inf

    def seed(self, dt_adm):
        self.dt_adm = dt_adm
        self.dt_new = self.forced_dt if self.forced_dt is not None else self.c_dt * dt_adm

    def next_dt(self):
        if self.forced_dt is not None:
            return self.forced_dt
        base = self.c_dt * self.dt_adm
        if self.averaging == "creeping":
            return 0.5 * (self.dt_old + base)
        return base

    def reset_for_rerun(self):
        if self.forced_dt is None:
            value = self.c_dt * self.dt_adm
            self.dt_old = value
            self.dt_new = value


def update_time_step_sizes(tc):
    """src/scheduler.py:77-85."""
    if not np.isfinite(tc.dt_adm) or tc.dt_adm <= 0.0:
        raise OracleError("NumericalError", f"admissible step degenerated to {tc.dt_adm}")
    tc.dt_old = tc.dt_new
    tc.dt_new = tc.next_dt()
    return tc.dt_new


# ---------------------------------------------------------------------------
# the fused driver (src/scheduler.py:92-449)

class FusedDriver:
    """Batched restatement of ``Driver(..., mode="fused")``.

    ``Q``: (n_cells,) + (n,)*d + (m,) float64 in reference cell order; it is
    updated in place like ``grid.cells[i].Q``.
    """

    def __init__(self, Q, d, p, L, cfl=DEFAULT_CFL, c_dt=DEFAULT_C_DT,
                 averaging="strict", forced_dt=None, inject_rerun=False,
                 spike_step=None, spike_factor=3.0, velocity=None, boundary="periodic"):
        """``velocity`` given: AdvectionSystem(d, velocity) (m = 1), else Euler."""
        pde = AdvectionPDE(d, velocity) if velocity is not None else EulerPDE(d)
        if velocity is not None and spike_step is not None:
            raise OracleError("ConfigurationError", "the speed spike is defined for Euler runs")
        self.k = OracleKernels(d, p, L, cfl, pde, boundary)
        self.d, self.p, self.L = d, p, L
        self.Q = Q
        self.D = np.zeros_like(Q)                       # src/mesh.py:238-239
        self.tc = TimeControl(c_dt, averaging, forced_dt)
        self.inject_rerun = inject_rerun
        self.spike_step, self.spike_factor = spike_step, spike_factor
        self.sweep_count = self.step_count = self.rerun_count = 0
        self.reruns_by_step = Counter()
        self.step_records = []
        self._primed = False
        self._tr = None           # traces of the last prediction pass
        self._seed_time_control()

    def _seed_time_control(self):
        """src/scheduler.py:135-155."""
        dt, ok, _ = self.k.calc_time_step(self.Q)
        if not np.all(ok):
            ci = int(np.nonzero(~ok)[0][0])
            raise OracleError("NumericalError", f"initial data inadmissible in cell {ci}", ci)
        adm = float(np.min(dt))
        if not np.isfinite(adm) or adm <= 0.0:
            raise OracleError("NumericalError", f"no admissible initial step (got {adm})")
        self.tc.seed(adm)

    def _predict_pass(self, dt, step, calc_fail=None):
        q, f, pfail, _ = self.k.predict(self.Q, dt)
        key = np.full(self.Q.shape[0], np.iinfo(np.int64).max, dtype=np.int64)
        cells = np.arange(self.Q.shape[0])
        if calc_fail is not None:
            key = np.where(calc_fail, 2 * cells, key)
            pfail = pfail & ~calc_fail
        key = np.where(pfail, np.minimum(key, 2 * cells + 1), key)
        kmin = int(key.min())
        if kmin != np.iinfo(np.int64).max:
            ci, phase = divmod(kmin, 2)
            if phase == 0:
                raise OracleError("NumericalError",
                                  f"inadmissible state in cell {ci} at step {step}", ci, step)
            raise OracleError("PredictorFailureError",
                              f"predictor produced non-finite values (cell {ci})", ci, step)
        self._tr = self.k.extrapolate(q, f)
        self.D = self.k.integrate_volume(f, dt)

    def _apply_spike(self):
        """src/scheduler.py:166-178."""
        d = self.d
        Q = self.Q
        rho = Q[..., 0]
        p = pressure(Q, d)
        j = Q[..., 1:1 + d] * self.spike_factor
        Q[..., 1:1 + d] = j
        Q[..., -1] = p / 0.4 + 0.5 * np.sum(j * j, axis=-1) / rho

    def _maybe_rerun(self, step):
        """src/scheduler.py:370-392."""
        tc = self.tc
        if not (self.inject_rerun or tc.dt_adm < tc.dt_old):
            return
        if self.reruns_by_step[step]:
            raise OracleError("NumericalError", f"second rerun requested within realisation step {step}")
        self.rerun_count += 1
        self.reruns_by_step[step] += 1
        tc.reset_for_rerun()
        self.sweep_count += 1
        self._predict_pass(tc.dt_old, step)
        if tc.forced_dt is None and tc.dt_adm < tc.dt_old:
            raise OracleError("NumericalError", "rerun failed to restore admissibility")

    def _sweep_fused(self, step):
        """src/scheduler.py:394-449."""
        k, tc = self.k, self.tc
        priming = step == 0
        if not priming:
            self._maybe_rerun(step)
        dt_old, dt_new = tc.dt_old, tc.dt_new
        self.sweep_count += 1
        if not priming:
            tr_q, tr_f = self._tr
            fstar = k.solve_riemann(tr_q, tr_f)
            self.D = k.integrate_face(self.D, fstar, dt_old)
        else:
            # never-populated hulls: F* = 0 and dt_old = 0 (src/kernels.py:158-163)
            self.D = self.D - 0.0
        self.Q += self.D                                   # src/kernels.py:213
        if self.spike_step is not None and step == self.spike_step:
            self._apply_spike()
        dt, ok, _ = k.calc_time_step(self.Q)
        adm = float(np.min(np.where(ok, dt, np.inf)))
        self._predict_pass(dt_new, step, calc_fail=~ok)
        if not priming:
            tc.T += dt_old
        tc.dt_adm = adm
        update_time_step_sizes(tc)

    def step(self):
        """src/scheduler.py:190-208."""
        if not self._primed:
            self._sweep_fused(0)
            self._primed = True
        self._sweep_fused(self.step_count + 1)
        self.step_count += 1
        tc = self.tc
        self.step_records.append({
            "step": self.step_count, "T": tc.T, "dt_old": tc.dt_old,
            "dt_new": tc.dt_new, "dt_adm": tc.dt_adm,
            "reruns": self.reruns_by_step[self.step_count], "troubled": 0})
        return self.step_count

    def run(self, steps):
        for _ in range(steps):
            self.step()
        return self.step_count


class StraightforwardDriver(FusedDriver):
    """Batched restatement of ``Driver(..., mode="straightforward")`` without
    limiter (src/scheduler.py:230-313): three phase-pure sweeps per step
    (predict + extrapolate; Riemann; volume + face + update + calc_time_step),
    step size ``dt = tc.dt_new`` of the previous step, no priming, no rerun."""

    def step(self):
        k, tc = self.k, self.tc
        step = self.step_count + 1
        dt = tc.dt_new
        q, f, pfail, _ = k.predict(self.Q, dt)                      # sweep 1
        if np.any(pfail):
            ci = int(np.nonzero(pfail)[0][0])
            raise OracleError("PredictorFailureError",
                              f"predictor produced non-finite values (cell {ci})", ci, step)
        tr_q, tr_f = k.extrapolate(q, f)
        fstar = k.solve_riemann(tr_q, tr_f)                         # sweep 2
        D = k.integrate_volume(f, dt)                               # sweep 3
        D = k.integrate_face(D, fstar, dt)
        self.Q += D
        if self.spike_step is not None and step == self.spike_step:
            self._apply_spike()
        dtc, ok, _ = k.calc_time_step(self.Q)
        if not np.all(ok):
            ci = int(np.nonzero(~ok)[0][0])
            raise OracleError("NumericalError", f"inadmissible state in cell {ci} at step {step}", ci, step)
        self.sweep_count += 3
        tc.T += dt
        tc.dt_adm = float(np.min(dtc))
        update_time_step_sizes(tc)
        self.step_count = step
        self.step_records.append({
            "step": step, "T": tc.T, "dt_old": tc.dt_old, "dt_new": tc.dt_new,
            "dt_adm": tc.dt_adm, "reruns": 0, "troubled": 0})
        return step
