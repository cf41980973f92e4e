"""CPU oracle of the a-posteriori subcell FV limiter — TEST INFRASTRUCTURE ONLY.

Only ``tests/`` (and the golden-vector tooling) may import this module; the
product path never does.  It restates, in batched numpy, the reference's
``SubcellLimiter`` (``src/limiter.py:26-234``) and the limiter branch of the
straightforward driver (``src/scheduler.py:230-313``), with
``src/`` = ``/root/reference/pkg/src/aderdg/``.

Semantics kept from the reference (they change results, so the GPU follows
them too):

* ``prev_Q`` is refreshed inside ``Kernels.update`` (``src/kernels.py:208-214``)
  cell by cell along the traversal, and the discrete-maximum-principle test of
  a cell runs right after its own update (``src/scheduler.py:282-284``).  So a
  face neighbour that precedes the cell in the traversal contributes its
  freshly snapshotted state (Q^n), a later one its snapshot of the step
  before (Q^(n-1); zeros before the first update, ``src/mesh.py:90-96``).
* ``troubled`` persists: it is set by a predictor failure (then the cell is
  re-predicted with dt = 0, ``src/scheduler.py:240-249``), by detection, or
  by an inadmissible corrected state, and cleared only by a successful
  reconstruction (``src/limiter.py:221-224``).
* troubled cells are re-advanced from their ``prev_Q`` by first-order
  Rusanov FV sub-steps on (2p+1)^d subcells, the neighbours' projected
  ``prev_Q`` as a frozen one-layer halo (``src/limiter.py:170-234``).

Pinning: ``tests/test_limiter_oracle.py`` compares this file against golden
runs of the reference itself (``tests/golden/make_limiter_golden.py``).
"""

import numpy as np

from aderdg_oracle import (OracleError, OracleKernels, TimeControl, apply_matrix,
                           lagrange_eval, update_time_step_sizes, StraightforwardDriver)

DMP_ABS = 1e-3      # src/limiter.py:23
DMP_REL = 1e-2      # src/limiter.py:24


def subcell_average_matrix(basis):
    """src/limiter.py:26-34: P[s, i] = mean of Lagrange polynomial i over
    subcell s of (0, 1) split into 2p+1 equal parts (Gauss quadrature)."""
    ns = 2 * basis.p + 1
    P = np.empty((ns, basis.n))
    for s in range(ns):
        P[s, :] = basis.weights @ lagrange_eval(basis.nodes, (s + basis.nodes) / ns)
    return P


def _take_layer(block, axis, index):
    """One-layer slab of ``block`` along ``axis`` (axis kept, size 1)."""
    return np.take(block, [index], axis=axis)


def rusanov_fv_step(states, h_sub, dt, pde, halo="periodic", cfl=0.9):
    """src/limiter.py:41-84: one first-order Godunov/Rusanov step on a block
    of subcell averages (no leading cell axis).  ``halo``: "periodic" or
    per-axis (low_slab, high_slab) one-layer slices."""
    d = states.ndim - 1
    lam = 0.0
    for axis in range(d):
        lam = max(lam, float(np.max(pde.max_signal_speed(states, axis))))
    if lam > 0.0 and dt > cfl * h_sub / (d * lam) * (1.0 + 1e-12):
        raise OracleError("NumericalError",
                          f"finite-volume step {dt} exceeds the admissible "
                          f"{cfl * h_sub / (d * lam)}; take a smaller step")
    out = states.copy()
    for axis in range(d):
        if isinstance(halo, str):
            low, high = _take_layer(states, axis, -1), _take_layer(states, axis, 0)
        else:
            low, high = halo[axis]
        ext = np.concatenate([low, states, high], axis=axis)
        n_ext = ext.shape[axis]
        left = np.take(ext, range(0, n_ext - 1), axis=axis)
        right = np.take(ext, range(1, n_ext), axis=axis)
        fl = pde.flux(left)[axis]
        fr = pde.flux(right)[axis]
        alpha = np.maximum(pde.max_signal_speed(left, axis),
                           pde.max_signal_speed(right, axis))[..., None]
        fstar = 0.5 * (fl + fr) - 0.5 * alpha * (right - left)
        n_if = fstar.shape[axis]
        out -= (dt / h_sub) * (np.take(fstar, range(1, n_if), axis=axis)
                               - np.take(fstar, range(0, n_if - 1), axis=axis))
    return out


class OracleLimiter:
    """src/limiter.py:87-234 over a periodic grid (leading cell axis)."""

    def __init__(self, k, cfl=0.9):
        b, d = k.basis, k.d
        self.k, self.pde, self.d = k, k.pde, d
        self.cfl = cfl
        self.ns = 2 * b.p + 1
        self.h_sub = k.h / self.ns
        self.P = subcell_average_matrix(b)
        self.R = np.linalg.solve(self.P.T @ self.P, self.P.T)     # src/limiter.py:99
        W = np.ones((b.n,) * d)
        for a in range(d):
            W = W * b.weights.reshape([b.n if c == a else 1 for c in range(d)])
        self.mean_weights = W[..., None]
        centers = (np.arange(self.ns) + 0.5) / self.ns
        self.nearest = np.argmin(np.abs(centers[:, None] - b.nodes[None, :]), axis=1)
        self.sample = np.minimum((b.nodes * self.ns).astype(int), self.ns - 1)

    # src/limiter.py:111-117 (one cell, no leading axis)
    def project(self, Q):
        for a in range(self.d):
            Q = apply_matrix(self.P, Q, a)
        return Q

    def admissible(self, Q):
        return bool(self.pde.admissible_per_cell(Q[None])[0])

    # src/limiter.py:119-134
    def reconstruct(self, patch):
        d = self.d
        Q = patch
        for a in range(d):
            Q = apply_matrix(self.R, Q, a)
        sp = tuple(range(d))
        Q = Q + (patch.mean(axis=sp) - np.sum(self.mean_weights * Q, axis=sp))
        return Q, self.admissible(Q) and self.admissible(self.project(Q))

    # src/limiter.py:138-160 (batched; prev = Q^n for cells at or before c in
    # the traversal, Q^(n-1) after it, see the module docstring)
    def detect(self, Q, cur, old, rank, cells=None):
        d, k = self.d, self.k
        C = Q.shape[0]
        sp = tuple(range(1, d + 1))
        with np.errstate(all="ignore"):
            ok = self.pde.admissible_per_cell(Q)
            patch = Q
            for a in range(d):
                patch = apply_matrix(self.P, patch, 1 + a)
            ok &= self.pde.admissible_per_cell(patch)
            cmin, cmax = cur.min(axis=sp), cur.max(axis=sp)
            omin, omax = old.min(axis=sp), old.max(axis=sp)
            lo, hi = cmin.copy(), cmax.copy()
            me = np.arange(C)
            for a in range(d):
                for nb in (k.minus[a], k.plus[a]):
                    there = (nb >= 0)[:, None]           # outflow: no neighbour (limiter.py:150-151)
                    nbc = np.where(nb >= 0, nb, me)
                    before = (rank[nbc] <= rank[me])[:, None]
                    lo = np.where(there, np.minimum(lo, np.where(before, cmin[nbc], omin[nbc])), lo)
                    hi = np.where(there, np.maximum(hi, np.where(before, cmax[nbc], omax[nbc])), hi)
            delta = DMP_ABS + DMP_REL * (hi - lo)
            cand_lo = np.minimum(Q.min(axis=sp), patch.min(axis=sp))
            cand_hi = np.maximum(Q.max(axis=sp), patch.max(axis=sp))
            dmp = np.any(cand_lo < lo - delta, axis=1) | np.any(cand_hi > hi + delta, axis=1)
        return ~ok | dmp

    # src/limiter.py:164-175
    def start_patch(self, Q):
        patch = self.project(Q)
        if self.admissible(patch):
            return patch
        for a in range(self.d):
            Q = np.take(Q, self.nearest, axis=a)
        return Q

    # src/limiter.py:177-194 + 196-234 for one troubled cell
    def apply_cell(self, ci, prev, dt):
        d, k = self.d, self.k
        patch = self.start_patch(prev[ci])
        halo = []
        for a in range(d):
            lo_nb, hi_nb = k.minus[a][ci], k.plus[a][ci]
            # outflow boundary: zero-gradient copy of the own edge (limiter.py:185-187)
            low = (_take_layer(self.start_patch(prev[lo_nb]), a, -1) if lo_nb >= 0
                   else _take_layer(patch, a, 0))
            high = (_take_layer(self.start_patch(prev[hi_nb]), a, 0) if hi_nb >= 0
                    else _take_layer(patch, a, -1))
            halo.append((low, high))
        remaining = dt
        while remaining > 1e-15 * dt:
            lam = 0.0
            for a in range(d):
                lam = max(lam, float(np.max(self.pde.max_signal_speed(patch, a))))
            dt_sub = remaining if lam <= 0.0 else min(remaining, self.cfl * self.h_sub / (d * lam))
            patch = rusanov_fv_step(patch, self.h_sub, dt_sub, self.pde, halo=halo, cfl=self.cfl)
            if not self.admissible(patch):
                raise OracleError("NumericalError",
                                  f"subcell update left cell {ci} inadmissible", ci)
            remaining -= dt_sub
        cand, ok = self.reconstruct(patch)
        if ok:
            return cand, False
        sampled = patch
        for a in range(d):
            sampled = np.take(sampled, self.sample, axis=a)
        return sampled, True


class LimitedStraightforwardDriver(StraightforwardDriver):
    """``Driver(..., "straightforward", limiter=SubcellLimiter(...))``
    (src/scheduler.py:230-313) with a traversal given as a permutation."""

    def __init__(self, Q, d, p, L, order=None, **kw):
        super().__init__(Q, d, p, L, **kw)
        C = Q.shape[0]
        self.order = np.arange(C) if order is None else np.asarray(order)
        self.rank = np.empty(C, dtype=np.int64)
        self.rank[self.order] = np.arange(C)
        self.lim = OracleLimiter(self.k, self.k.cfl)
        self.cur = np.zeros_like(Q)          # prev_Q after this step's update (Q^n)
        self.old = np.zeros_like(Q)          # prev_Q of the step before (src/mesh.py:90-96)
        self.troubled = np.zeros(C, dtype=bool)
        self.troubled_by_step = {}

    def _first(self, mask):
        return int(self.order[np.argmax(mask[self.order])])

    def step(self):
        k, tc = self.k, self.tc
        step = self.step_count + 1
        dt = tc.dt_new
        q, f, pfail, _ = k.predict(self.Q, dt)                        # sweep 1
        if np.any(pfail):
            C = self.Q.shape[0]
            finite = np.all(np.isfinite(self.Q.reshape(C, -1)), axis=1)
            idx = np.nonzero(pfail)[0]
            with np.errstate(all="ignore"):
                q0, f0, fail0, _ = k.predict(self.Q[idx], 0.0)   # the retry of scheduler.py:246
            bad = np.zeros(C, dtype=bool)
            bad[idx[fail0]] = True                 # includes non-finite Q (kernels.py:80-81)
            bad |= pfail & ~finite
            if np.any(bad):
                ci = self._first(bad)
                raise OracleError("PredictorFailureError",
                                  f"predictor produced non-finite values (cell {ci})", ci, step)
            q[idx], f[:, idx] = q0, f0
            self.troubled[idx] = True
        tr_q, tr_f = k.extrapolate(q, f)
        fstar = k.solve_riemann(tr_q, tr_f)                           # sweep 2
        D = k.integrate_volume(f, dt)                                 # sweep 3
        D = k.integrate_face(D, fstar, dt)
        self.old, self.cur = self.cur, self.Q.copy()                  # Kernels.update snapshot
        self.Q += D
        if self.spike_step is not None and step == self.spike_step:
            self._apply_spike()
        self.troubled |= self.lim.detect(self.Q, self.cur, self.old, self.rank)
        dtc, ok, _ = k.calc_time_step(self.Q)
        self.troubled |= ~ok
        adm = np.where(ok, dtc, np.inf)
        n_troubled = int(np.count_nonzero(self.troubled))
        if n_troubled:                                                # src/scheduler.py:301-309
            self.troubled_by_step[step] = n_troubled
            limited = self.troubled.copy()
            for ci in self.order[limited[self.order]]:
                self.Q[ci], self.troubled[ci] = self.lim.apply_cell(int(ci), self.cur, dt)
            tv, tok, _ = k.calc_time_step(self.Q)
            adm = np.where(limited, np.where(tok, tv, np.inf), adm)
        self.sweep_count += 3
        tc.T += dt
        tc.dt_adm = float(np.min(adm))
        update_time_step_sizes(tc)
        self.step_count = step
        self.step_records.append({
            "step": step, "T": tc.T, "dt_old": tc.dt_old, "dt_new": tc.dt_new,
            "dt_adm": tc.dt_adm, "reruns": 0, "troubled": n_troubled})
        return step
