"""Access accounting of the GPU drivers, in the reference's units.

The reference books every kernel-task invocation on an ``AccessLedger``
(``src/metrics.py:108-186``): logical doubles read/written per task, the
"bus model" blocks per task, and the Q_h fetch counter, each attributed to a
realisation step.  On the GPU a sweep is one kernel over all cells, so the
counts are not observed per call; they follow exactly from the driver's
schedule, which is fixed by (mode, d, p, m, cells, faces) and the rerun
decisions the device reports.  ``AccessLedger.book_*`` adds them per sweep with
the reference's attribution rules, so ``metrics.csv`` and ``run.json`` carry
the same integers the reference writes for the same run.

Per-cell trace events (``TraceEvent``, ``validate_trace``) describe the CPU
scheduler's sequential task order; the GPU has no such order inside a sweep
and does not produce them.

Reference citations (``src/`` = ``/root/reference/pkg/src/aderdg/``):
  TASKS / STP_TASKS               src/metrics.py:25-30
  logical_task_volumes            src/metrics.py:47-61
  _bus_profile                    src/metrics.py:64-99
  AccessLedger._record            src/metrics.py:157-175
  persistent_footprint ... audit  src/metrics.py:191-278
"""

from collections import Counter
from fractions import Fraction

from .errors import ConfigurationError

TASKS = ("predict", "extrapolate", "solveRiemann", "integrateVolume",
         "integrateFace", "update", "calcTimeStep")
STP_TASKS = frozenset({"predict", "extrapolate", "integrateVolume"})
MODES = ("straightforward", "shifted", "fused")


def logical_task_volumes(task, d, p, m):
    """(reads, writes) in doubles for one invocation of a kernel task."""
    n = p + 1
    block = m * n ** d
    st = m * n ** (d + 1)
    table = {
        "predict": (block, (d + 1) * st),
        "extrapolate": ((d + 1) * st, 4 * d * block),
        "solveRiemann": (4 * block, 2 * block),
        "integrateVolume": (d * st, block),
        "integrateFace": (2 * d * block, block),
        "update": (block, block),
        "calcTimeStep": (block, 1),
    }
    return table[task]


def bus_profile(mode, d):
    """Blocks of m(p+1)^d doubles (read, written) per task invocation under the
    reference's cache model: straightforward (18d+4), fused (16d+3) plus
    (4d+2) per rerun pass."""
    if mode == "straightforward":
        return {"predict": (1, 1), "extrapolate": (0, 4 * d), "solveRiemann": (8, 4),
                "integrateVolume": (0, 0), "integrateFace": (2 * d, 0), "update": (1, 1),
                "calcTimeStep": (0, 0)}
    if mode == "shifted":
        return {"predict": (1, 0), "extrapolate": (0, 4 * d), "solveRiemann": (8, 4),
                "integrateVolume": (0, 1), "integrateFace": (2 * d + 1, 0), "update": (1, 1),
                "calcTimeStep": (0, 0)}
    if mode == "fused":
        return {"predict": (0, 0), "extrapolate": (0, 4 * d), "solveRiemann": (8, 4),
                "integrateVolume": (0, 1), "integrateFace": (1, 0), "update": (0, 1),
                "calcTimeStep": (0, 0)}
    raise ConfigurationError(f"unknown scheduler mode {mode!r}")


class AccessLedger:
    """Closed-form counterpart of the reference ledger.  The driver calls
    ``begin_sweep`` with the reference's (completing, predicting, rerun_pass)
    context and then ``book(task, count)`` once per task kind with the number of
    entities the sweep touched."""

    def __init__(self, mode, d, p, m, trace_enabled=False):
        if mode not in MODES:
            raise ConfigurationError(f"unknown scheduler mode {mode!r}")
        if trace_enabled:
            raise ConfigurationError(
                "per-task traces describe the CPU scheduler's sequential order; "
                "the GPU runs each sweep as one kernel and records none")
        self.mode = mode
        self.d, self.p, self.m = d, p, m
        self.block = m * (p + 1) ** d
        self.task_invocations = Counter()
        self.task_reads = Counter()
        self.task_writes = Counter()
        self.bus_reads_by_step = Counter()
        self.bus_writes_by_step = Counter()
        self.q_reads_by_step = Counter()
        self.trace = []
        self.trace_enabled = False
        self._profile = bus_profile(mode, d)
        self._completing = 0
        self._predicting = 0
        self._rerun_pass = False

    def begin_sweep(self, sweep, completing_step, predicting_step, rerun_pass=False):
        self._completing = completing_step
        self._predicting = predicting_step
        self._rerun_pass = rerun_pass

    def book(self, task, count):
        """``count`` invocations of ``task`` in the current sweep
        (src/metrics.py:157-175 applied ``count`` times)."""
        step = self._predicting if task in STP_TASKS else self._completing
        r, w = logical_task_volumes(task, self.d, self.p, self.m)
        self.task_invocations[task] += count
        self.task_reads[task] += r * count
        self.task_writes[task] += w * count
        br, bw = self._profile[task]
        if self._rerun_pass and task == "predict":
            br = 1
        self.bus_reads_by_step[step] += br * self.block * count
        self.bus_writes_by_step[step] += bw * self.block * count
        if task == "update":
            self.q_reads_by_step[step] += count
        elif task == "predict" and (self.mode != "fused" or self._rerun_pass):
            self.q_reads_by_step[step] += count

    def step_traffic(self, step):
        return self.bus_reads_by_step[step], self.bus_writes_by_step[step]

    def total_traffic(self, first_step, last_step):
        reads = sum(self.bus_reads_by_step[s] for s in range(first_step, last_step + 1))
        writes = sum(self.bus_writes_by_step[s] for s in range(first_step, last_step + 1))
        return reads + writes


def book_fused_sweep(ledger, sweep, step, cells, faces):
    """One regular fused sweep (src/scheduler.py:394-449): completes ``step``,
    predicts ``step + 1``; every face solved once, every cell corrected and
    re-predicted."""
    ledger.begin_sweep(sweep, step, step + 1)
    ledger.book("solveRiemann", faces)
    for t in ("integrateFace", "update", "calcTimeStep", "predict", "extrapolate",
              "integrateVolume"):
        ledger.book(t, cells)


def book_rerun_pass(ledger, sweep, step, cells):
    """The rerun prediction pass of ``step`` (src/scheduler.py:370-392)."""
    ledger.begin_sweep(sweep, step - 1, step, rerun_pass=True)
    for t in ("predict", "extrapolate", "integrateVolume"):
        ledger.book(t, cells)


def book_straightforward_step(ledger, sweep, step, cells, faces, troubled=0):
    """The three sweeps of a straightforward step (src/scheduler.py:230-313); with a
    limiter every troubled cell books one more calcTimeStep after its subcell
    pass (src/scheduler.py:307-309; the limiter itself records nothing)."""
    ledger.begin_sweep(sweep, step, step)
    ledger.book("predict", cells)
    ledger.book("extrapolate", cells)
    ledger.begin_sweep(sweep + 1, step, step)
    ledger.book("solveRiemann", faces)
    ledger.begin_sweep(sweep + 2, step, step)
    for t in ("integrateVolume", "integrateFace", "update", "calcTimeStep"):
        ledger.book(t, cells)
    if troubled:
        ledger.book("calcTimeStep", troubled)


def record_step(ledger, mode, step, reruns, cells, faces, troubled=0):
    """Book realisation step ``step`` of a GPU run (priming sweep inside step 1,
    the rerun pass when ``reruns``) and return the ledger columns of its
    metrics record, as ``Driver._record_step`` does (src/scheduler.py:459-481)."""
    reads0, writes0 = Counter(ledger.task_reads), Counter(ledger.task_writes)
    if mode == "straightforward":
        book_straightforward_step(ledger, 3 * (step - 1), step, cells, faces, troubled)
    else:
        if step == 1:
            book_fused_sweep(ledger, 0, 0, cells, faces)
        if reruns:
            book_rerun_pass(ledger, -1, step, cells)
        book_fused_sweep(ledger, -1, step, cells, faces)
    rec = {}
    for task in ledger.task_reads.keys() | reads0.keys():
        rec[f"{task}_reads"] = ledger.task_reads[task] - reads0[task]
        rec[f"{task}_writes"] = ledger.task_writes[task] - writes0[task]
    rec["q_reads_per_cell"] = ledger.q_reads_by_step[step] / cells
    rec["bus_reads"] = ledger.bus_reads_by_step[step]
    rec["bus_writes"] = ledger.bus_writes_by_step[step]
    return rec


# ---------------------------------------------------------------------------
# closed-form models (src/metrics.py:191-242)

def persistent_footprint(mode, d, p, m):
    n = p + 1
    block = m * n ** d
    if mode in ("fused", "shifted"):
        return (2 + 6 * d) * block
    if mode == "straightforward":
        return (d + 1) * m * n ** (d + 1) + (1 + 6 * d) * block
    raise ConfigurationError(f"unknown scheduler mode {mode!r}")


def footprint_ratio(d, p):
    if d not in (2, 3):
        raise ConfigurationError(f"dimension must be 2 or 3, got {d}")
    if not 0 <= p <= 9:
        raise ConfigurationError(f"order p must be in [0, 9], got {p}")
    return Fraction(2 + 6 * d, (d + 1) * (p + 1) + 1 + 6 * d)


def traffic_model(mode, d, p, m, c_rerun=1.0):
    if not 1.0 <= c_rerun <= 2.0:
        raise ConfigurationError(f"c_rerun must be in [1, 2], got {c_rerun}")
    block = m * (p + 1) ** d
    if mode == "straightforward":
        return (18 * d + 4) * block
    if mode == "fused":
        return ((4 * d + 2) * c_rerun + 12 * d + 1) * block
    if mode == "shifted":
        return (18 * d + 5) * block
    raise ConfigurationError(f"unknown scheduler mode {mode!r}")


def rerun_upper_bound(t_3steps, t_stp, t_fused, c_dt):
    if not (0 < t_stp < t_3steps and t_fused > 0):
        raise ConfigurationError("need 0 < T_stp < T_3steps and T_fused > 0")
    return 1.0 + (t_3steps * c_dt - t_fused) / t_stp


def single_touch_audit(ledger, n_cells, steps):
    per_step = {s: ledger.q_reads_by_step[s] / n_cells for s in range(1, steps + 1)}
    total = sum(ledger.q_reads_by_step[s] for s in range(1, steps + 1))
    return {"per_step": per_step, "amortised": total / (n_cells * steps),
            "total_q_reads": total}


def traffic_audit(ledger, n_cells, steps, c_rerun=1.0):
    model = traffic_model(ledger.mode, ledger.d, ledger.p, ledger.m, c_rerun)
    per_step = {}
    total = 0
    for s in range(1, steps + 1):
        r, w = ledger.step_traffic(s)
        per_step[s] = r + w
        total += r + w
    return {"per_step": per_step, "measured_per_cell_step": total / (n_cells * steps),
            "model_per_cell_step": model, "total": total}


def estimate_persistent_doubles(d, L, p, m, boundary="periodic", storage="hull"):
    """src/mesh.py:149-164: the reference's allocation count for a grid (the
    run.json ``persistent_doubles`` figure)."""
    n = p + 1
    cells = 3 ** (d * L)
    per_axis = 3 ** L
    n_faces = d * cells if boundary == "periodic" else d * (per_axis + 1) * per_axis ** (d - 1)
    block = n ** d * m
    total = cells * n ** d * m
    if storage == "hull":
        total += cells * n ** d * m
    else:
        total += cells * (d + 1) * m * n ** (d + 1)
    total += n_faces * 6 * block
    return total
