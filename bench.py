#!/usr/bin/env python
"""bench.py — fp64 DoF-updates/s of the fused ADER-DG Euler step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

Metric (BASELINE.json): fp64 DoF-updates/s for 3D Euler ADER-DG at order p on
1/2/4/8 B200, DoF = cells * (p+1)^d * m.  Default workload = BASELINE config 4,
the configuration the metric is quoted on at 1/2/4/8 GPUs: 3D Euler p=5 on the
81^3 periodic grid (531441 cells, 5.74e8 DoF), Gaussian bump + seeded 1e-3
density noise, Rusanov, CFL 0.9/(d(2p+1)), c_dt 0.99.  A "step" is one fused
realisation step of the whole grid (rerun pass when the optimistic step fails,
fused Riemann/corrector/update/CFL/predictor sweep, device time control).
``--config`` selects the other BASELINE configurations (parity-test cases and
per-order measurements).

GPUs: one process per GPU.  Under torchrun (WORLD_SIZE set) this process is one
rank; ``--gpus N > 1`` without torchrun launches the N ranks itself through
``torch.distributed.run`` and fails loudly when fewer than N GPUs are visible.
N > 1: x-slab decomposition of the fixed grid (strong scaling), NCCL halo
exchange of the slab-boundary face records hidden behind the interior planes,
MAX all-reduce of the step reduction, the steps of a segment enqueued from C as
one CUDA graph over the library's own NCCL communicator.  NCCL's INIT log goes
to stderr (NCCL_DEBUG=INFO, NCCL_DEBUG_SUBSYS=INIT) so the rank count is visible.

Reported on one JSON line (rank 0):
  value         DoF-updates/s, device-timed (CUDA events on the launch stream around
                the timed steps, max over ranks), state resident in HBM
  e2e           same metric through the C ABI with host buffers: per step pinned H2D of
                the state, the step, D2H of the state (wall clock, max over ranks)
  roofline      the sweep kernel (fused sweep + rerun passes): algorithmic flops
                (paper_1801_08682_b200/roofline.py with the measured Picard counts) per
                step / its time per step, against the measured FP64 peak
                (profiles/fp64_peaks_r02.jsonl; MEASURED_PEAKS.json has no fp64 entry)
  cpu_baseline  the CPU oracle port (oracle/aderdg_oracle.py, batched numpy restatement of
                the reference fused driver) on ONE pinned host core, plus a row with all
                host cores as BLAS threads; per-cell-step cost measured on a 9^3 sample of
                the same state family, times the workload's cells (labelled extrapolated)
--impl reference: the same oracle port with all host cores on the same config, metric and
unit (rank 0 only; other ranks exit 0).  The reference package is CPU-only Python that
cannot travel to the GPU box; its oracle restatement is pinned to it by tests/golden.
"""

import argparse
import ctypes
import json
import os
import socket
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    "cfg1": dict(d=2, L=3, p=3, scenario="bump", steps=20,
                 desc="BASELINE cfg1: 2D Euler p=3, 27^2 periodic, bump+1e-3 noise, 20 steps"),
    "cfg2": dict(d=3, L=3, p=3, scenario="bump", steps=20,
                 desc="BASELINE cfg2: 3D Euler p=3, 27^3 periodic, bump+1e-3 noise, 20 steps"),
    "cfg3_p5": dict(d=3, L=3, p=5, scenario="bump", steps=10,
                    desc="BASELINE cfg3: 3D Euler p=5, 27^3 periodic, bump+1e-3 noise, 10 steps"),
    # p = 7 / 9 with the specified noise blow up in the reference itself (NumericalError at
    # step 7 / step 5): timed on the steps before the abort
    "cfg3_p7": dict(d=3, L=3, p=7, scenario="bump", steps=6,
                    desc="BASELINE cfg3: 3D Euler p=7, 27^3 periodic, bump+1e-3 noise (6 pre-abort steps)"),
    "cfg3_p9": dict(d=3, L=3, p=9, scenario="bump", steps=4,
                    desc="BASELINE cfg3: 3D Euler p=9, 27^3 periodic, bump+1e-3 noise (4 pre-abort steps)"),
    # 81^3 p=5 with the specified noise aborts at step 10 (NumericalError, cell 208997; the
    # same instability the reference shows at 27^3 for p >= 7): timed in 9-step episodes
    "cfg4": dict(d=3, L=4, p=5, scenario="bump", steps=9,
                 desc="BASELINE cfg4: 3D Euler p=5, 81^3 periodic, bump+1e-3 noise (9-step episodes)"),
    "cfg5": dict(d=3, L=4, p=9, scenario="fourier", steps=5,
                 desc="BASELINE cfg5: 3D Euler p=9, 81^3 periodic, random Fourier state, 5 steps"),
}
DEFAULT_CONFIG = "cfg4"

PEAKS_FILE = os.path.join(REPO, "profiles", "fp64_peaks_r02.jsonl")
NCU_TRAFFIC_FILE = os.path.join(REPO, "profiles", "r02", "sweep_traffic.json")
METRIC = "fp64 DoF-updates/s (3D Euler ADER-DG, fused step)"


def load_peaks():
    dmma = dfma = None
    try:
        with open(PEAKS_FILE) as fh:
            for line in fh:
                r = json.loads(line)
                if r.get("test") == "dfma":
                    dfma = max(dfma or 0, r["tflops"])
                if r.get("test", "").startswith("dmma"):
                    dmma = max(dmma or 0, r["tflops"])
    except OSError:
        pass
    hbm = None
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            hbm = json.load(fh).get("hbm_gbs")
    except OSError:
        pass
    return dfma, dmma, hbm


def config_dict(name, cfgd, world, mode):
    """The workload description both arms print (identical for the same arguments)."""
    from paper_1801_08682_b200 import roofline
    d, L, p = cfgd["d"], cfgd["L"], cfgd["p"]
    cells = 3 ** (d * L)
    return {"workload": cfgd["desc"], "name": name, "d": d, "p": p, "L": L, "cells": cells,
            "nodes": cells * (p + 1) ** d, "dof": roofline.dof(d, p, cells), "driver": mode,
            "episode_steps": cfgd["steps"],
            "parallelism": f"x-slab x{world}" if world > 1 else "single GPU",
            "l2": "no flush: per-step working set (Q,D r/w + 2 trace parities) "
                  f"{roofline.bytes_step(d, p, cells) / 1e6:.0f} MB > 126 MB L2"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/adg_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm = float(parts[1])
                    mx = float(parts[2])
                except ValueError:
                    continue
                sms.append(sm)
                maxs.append(mx)
                for nm, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        if not sms:
            return None
        busy = [s for s in sms if s > 500] or sms
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(maxs),
                "samples": len(sms), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port of the reference fused driver
def cpu_port_rows(cfgd, steps, rows):
    """Median step time of the oracle port (oracle/aderdg_oracle.py) on a sample of the
    workload's state family: the full grid in 2D, a 9^3 grid in 3D (the port, like the
    reference's per-cell loop, costs the same per cell step at any grid size; 81^3 does not
    fit host memory).  ``rows``: [(label, BLAS threads, pinned core or None)], measured
    one after another on the same primed driver (steps after priming + 1 warm-up step,
    episodes restarted at the configured step count).  Returns per row
    (label, threads, core, per-cell-step seconds, step times)."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import aderdg_oracle as O
    from threadpoolctl import threadpool_limits
    from paper_1801_08682_b200 import scenarios
    d, p = cfgd["d"], cfgd["p"]
    Ls = cfgd["L"] if d == 2 else 2
    cells = 3 ** (d * Ls)
    E = cfgd["steps"]
    Q0 = scenarios.build(cfgd["scenario"], d, Ls, p)
    out = []
    affinity = os.sched_getaffinity(0)
    drv, done = None, 0
    for label, threads, core in rows:
        if core is not None:
            os.sched_setaffinity(0, {core})
        times = []
        try:
            with threadpool_limits(threads):
                while len(times) < steps:
                    if drv is None or done >= E:
                        drv, done = O.FusedDriver(Q0.copy(), d, p, Ls), 0
                        drv.step()            # priming sweep + step 1 (untimed)
                        done = 1
                    if not times:
                        drv.step()            # warm-up under this row's threads
                        done += 1
                        if done >= E:
                            continue
                    t0 = time.perf_counter()
                    drv.step()
                    times.append(time.perf_counter() - t0)
                    done += 1
        finally:
            os.sched_setaffinity(0, affinity)
        out.append((label, threads, core, statistics.median(times) / cells, times))
    return out, cells, Ls


def cpu_baseline_block(cfgd, steps, all_rows):
    from paper_1801_08682_b200 import roofline
    d, L, p = cfgd["d"], cfgd["L"], cfgd["p"]
    nproc = len(os.sched_getaffinity(0))
    core = max(os.sched_getaffinity(0))
    rows = [("1 pinned core", 1, core)]
    if all_rows:
        rows.append((f"{nproc} cores (BLAS threads)", nproc, None))
    res, cells_s, Ls = cpu_port_rows(cfgd, steps, rows)
    dof_cell = roofline.dof(d, p, 1)
    cells = 3 ** (d * L)
    extrap = cells_s != cells
    table = [{"label": lab, "cores": thr, "pinned_core": c, "value": dof_cell / cost,
              "sec_per_cell_step": cost, "steps_timed": len(ts)} for lab, thr, c, cost, ts in res]
    sample = (f"oracle/aderdg_oracle.py (batched numpy port of the reference fused driver, pinned to it "
              f"by tests/golden), {3 ** Ls}^{d} cells p={p} sample, median of {len(res[0][4])} steps after "
              f"priming + 1 warm-up step; "
              + (f"extrapolated to {3 ** L}^{d} cells by the per-cell-step cost" if extrap else "full grid")
              + f"; host nproc {nproc}")
    return table, sample, nproc


def run_reference(args, cfgd):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    table, sample, nproc = cpu_baseline_block(cfgd, args.steps, all_rows=True)
    # value: the faster of the two rows (all host cores as BLAS threads is not always faster
    # than one pinned core for the batched port)
    allc = max(table, key=lambda r: r["value"])
    line = {
        "impl": "reference", "metric": METRIC,
        "value": allc["value"], "unit": "DoF-updates/s", "n_gpus": world, "steps": allc["steps_timed"],
        "warmup": args.warmup, "ms_per_step": 1e3 * allc["sec_per_cell_step"] * 3 ** (cfgd["d"] * cfgd["L"]),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args.config, cfgd, world, args.mode),
        "cpu_baseline": {"value": allc["value"], "unit": "DoF-updates/s", "cores": allc["cores"],
                         "kind": "port", "sample": sample, "rows": table},
        "e2e": {"value": allc["value"], "unit": "DoF-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def launch_ranks(args):
    """--gpus N > 1 outside torchrun: start the N ranks through torch.distributed.run."""
    import torch
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if have < args.gpus:
        print(f"[bench] --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}", file=sys.stderr)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: one episode of the config minus the warm-up)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="fused", choices=["fused", "straightforward"],
                    help="driver: fused single-touch (north star) or the straightforward passes")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfgd = CONFIGS[args.config]
    if args.steps is None:
        args.steps = max(1, cfgd["steps"] - args.warmup)
    if args.impl == "reference":
        return run_reference(args, cfgd)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return launch_ranks(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1801_08682_b200 import _lib, roofline, scenarios
    from paper_1801_08682_b200.parallel import SlabDriver

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # ADG_BENCH_GLOO=1: every rank on cuda:0 with host-staged gloo transport -- a
    # functional check of the multi-rank code path on a one-GPU box (no timing claim)
    staged = os.environ.get("ADG_BENCH_GLOO") == "1" and world > 1
    if world != args.gpus:
        print(f"[bench] WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if not torch.cuda.is_available() or (not staged and torch.cuda.device_count() <= local):
        print(f"[bench] rank {rank}: no CUDA device for local rank {local}", file=sys.stderr)
        return 2
    if staged:
        local = 0
    if world > 1 and not staged:
        # NCCL's INIT lines (comm nranks, rank -> device) on stderr, not on the JSON stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if staged:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    d, L, p = cfgd["d"], cfgd["L"], cfgd["p"]
    cells = 3 ** (d * L)
    dofs = roofline.dof(d, p, cells)
    Q0 = scenarios.build(cfgd["scenario"], d, L, p)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if staged else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- device-resident timing (value) ----------------
    # The seeded noisy BASELINE states are only integrated for the configured
    # number of steps E (the reference itself blows up past them at p >= 5,
    # SURVEY.md §7); longer timings restart episodes from Q0 outside the timed
    # segments.  Default K + W = E: one episode, the first W steps (incl. the
    # priming sweep) untimed.
    E = cfgd["steps"]
    drv = SlabDriver(Q0, d, L, p, rank, world, local, mode=args.mode, staged=staged)
    h = drv.handle
    # N > 1: the timed steps are enqueued from C over the library's own NCCL communicator
    native = world > 1 and not staged
    if native:
        drv.init_native_comm()
    K = args.steps
    clocks = ClockSampler(local)
    rerun_launches = []

    def timed_segments(flags):
        """Run K timed steps in episodes; returns (segment ms list, kernel ms, records)."""
        seg, kern, recs = [], 0.0, []
        rerun_launches.clear()
        remaining, first, started = K, True, False
        while remaining > 0:
            drv.load(Q0)                  # every episode restarts from the seeded state
            warm = args.warmup if first else 1
            for _ in range(warm):
                drv.enqueue_step()
            h.call("adg_sync")
            s0 = h.lib.adg_step_count(h.h)
            n = min(remaining, max(1, E - warm))
            barrier()
            torch.cuda.synchronize()
            if flags == 0 and not started:
                clocks.start()
                started = True
                time.sleep(0.05)
            if world == 1 or native:
                # the n steps back to back from C as one CUDA graph, CUDA events around the
                # segment (flags 0) or also around every rerun / sweep launch (replay)
                tout = (ctypes.c_double * 2)()
                if world == 1:
                    h.call("adg_run_timed_ex", n, flags, tout)
                else:
                    tout[0], tout[1] = drv.run_timed(n, flags=flags)
                seg.append(tout[0])
                kern += tout[1]
            else:
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                ev[0].record()
                for _ in range(n):
                    drv.enqueue_step()
                ev[1].record()
                torch.cuda.synchronize()
                seg.append(ev[0].elapsed_time(ev[1]))
            barrier()
            h.call("adg_sync")
            seg_recs = h.step_records(s0 + 1, n)
            recs += seg_recs
            # rerun-pass launches: the segment's first step (its conditional node defaults to
            # 1; the pass checks the rerun flag itself) and every later step that reruns
            rerun_launches.append(1 + sum(1 for r in seg_recs[1:] if r.reruns))
            remaining -= n
            first = False
        return seg, kern, recs

    seg_ms, _, recs = timed_segments(0)
    timed_rerun_launches = sum(rerun_launches)
    clk = clocks.stop()
    # instrumented replay of the same segments (same initial states, same launches) with
    # CUDA events around every rerun / sweep launch: the sweep kernel's share of the step
    rep_seg, rep_kern, rep_recs = timed_segments(_lib.ADG_TIMED_KERNEL_EVENTS) if (world == 1 or native) \
        else (seg_ms, 0.0, recs)
    elapsed_ms = max_over_ranks(sum(seg_ms))
    ms_per_step = elapsed_ms / K
    value = dofs * K / (elapsed_ms * 1e-3)
    iters = sum(r.picard_iters for r in recs)
    preds = sum(r.predicts for r in recs)
    reruns = sum(r.reruns for r in recs)
    local_cells = drv.n_local
    # per-step algorithmic flops of this rank: K steps of corrector work + the counted
    # Picard iterations / predicts of those steps
    flops_total = roofline.flops_step(d, p, local_cells * K, iters, preds)
    # 2D p = 3 on one GPU (cfg 1): each timed segment is ONE cooperative launch of
    # run_kernel_2d_p3 (sweeps, grid barriers and time control of all its steps): the kernel's
    # duration is the segment's, and the per-launch replay (the step graph) does not describe it
    multi_step = world == 1 and d == 2 and p == 3 and args.mode == "fused"
    share = (rep_kern / sum(rep_seg)) if (rep_kern > 0 and not multi_step) else None
    own_ms_per_step = sum(seg_ms) / K
    kern_ms_per_step = (share * own_ms_per_step) if share else own_ms_per_step
    achieved_tf = (flops_total / K) / (kern_ms_per_step * 1e-3) / 1e12
    achieved_tf = max_over_ranks(-achieved_tf) * -1 if world > 1 else achieved_tf   # slowest rank
    dfma, dmma, hbm = load_peaks()
    peak_tf = dmma or dfma or 37.1
    # ncu DRAM bytes of one full sweep launch (profiles/r02/sweep_traffic.json) x the sweep
    # passes per timed step (1 + the share of steps that rerun), like `achieved`
    traffic = traffic_launch = None
    try:
        with open(NCU_TRAFFIC_FILE) as fh:
            t = json.load(fh).get(args.config)
        if t and world == 1:
            traffic_launch = t["dram_bytes_per_step"] / t["full_sweep_launches_per_step"]
            traffic = traffic_launch * preds / (local_cells * K)
    except (OSError, ValueError, KeyError, ZeroDivisionError):
        pass
    bytes_alg = roofline.bytes_step(d, p, local_cells, preds // K)
    hbm_frac = (bytes_alg / (kern_ms_per_step * 1e-3) / 1e9) / hbm if hbm else None

    # ---------------- end-to-end through the C ABI with host buffers ----------------
    e2e = None
    if not args.no_e2e:
        n_state = int(drv.lay.state_doubles)
        pinned = torch.empty(n_state, dtype=torch.float64, pin_memory=True)
        hostQ = pinned.numpy()
        ptr = _lib.dptr(hostQ)
        e2e_s, remaining, first = 0.0, K, True
        while remaining > 0:
            drv.load(Q0)
            if world == 1:
                # warm-up through the same C-ABI call as the timed steps (its copy
                # streams, events and pinned record slot are created on first use)
                hostQ[:] = drv.local_state().reshape(-1)
                for _ in range(args.warmup if first else 1):
                    h.call("adg_step_host", ptr, ptr, None)
            else:
                for _ in range(args.warmup if first else 1):
                    drv.enqueue_step()
                hostQ[:] = drv.local_state().reshape(-1)
            n = min(remaining, max(1, E - (args.warmup if first else 1)))
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(n):
                if world == 1:
                    # H2D of the step's input, the step, D2H of its result, pipelined
                    # over plane chunks inside one C-ABI call (adg_step_host)
                    h.call("adg_step_host", ptr, ptr, None)
                else:
                    h.call("adg_load_state", ptr, n_state)   # H2D of the step's input state
                    drv.enqueue_step()
                    h.call("adg_store_state", ptr, n_state)  # D2H of the step's result (synchronous)
            t1 = time.perf_counter()
            barrier()
            e2e_s += t1 - t0
            h.call("adg_sync")
            remaining -= n
            first = False
        e2e_s = max_over_ranks(e2e_s)
        e2e = {"value": dofs * K / e2e_s, "unit": "DoF-updates/s",
               "h2d_bytes_per_step": 8 * n_state * world, "d2h_bytes_per_step": 8 * n_state * world,
               "ms_per_step": 1e3 * e2e_s / K,
               "path": ("adg_step_host: pinned H2D + fused step + D2H per step, pipelined over "
                        "wave-aligned cell chunks" if world == 1 else
                        "adg_load_state (pinned H2D) + overlapped slab step + adg_store_state (D2H), per step")}

    # our kernels launched in the timed steps: per step the sweep (two launches, interior and
    # boundary planes, on N > 1) and the time control; the rerun pass only where its
    # conditional node fires (a segment's first step, whose condition defaults to 1, and
    # steps after a finish that asked for a rerun)
    sweeps = 2 if (world > 1 and drv.lay.planes_local > 2) else 1
    launches = len(seg_ms) if multi_step else timed_rerun_launches + K * (sweeps + 1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        table, sample, nproc = cpu_baseline_block(cfgd, 2, all_rows=True)
        cpu = {"value": table[0]["value"], "unit": "DoF-updates/s", "cores": 1, "kind": "port",
               "sample": sample, "host_nproc": nproc, "rows": table}

    if rank == 0:
        conf = config_dict(args.config, cfgd, world, args.mode)
        conf["exchange"] = (None if world == 1 else "gloo staged (functional only)" if staged
                            else "library NCCL comm, steps enqueued from C as one CUDA graph")
        line = {
            "metric": METRIC,
            "value": value, "unit": "DoF-updates/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": conf,
            "run": {"episodes": len(seg_ms), "reruns_in_timed": reruns,
                    "picard_mean": iters / max(preds, 1), "predicts": preds, "picard_iters": iters},
            # compute-bound on the FP64 datapath; the peak is the measured FP64 tensor-core
            # (DMMA) throughput, which the CUDA-core DFMA pipe shares (contract: hbm | tensor)
            "roofline": {"bound": "tensor", "datapath": "fp64 (DMMA m8n8k4 + DFMA)",
                         "achieved": achieved_tf, "peak": peak_tf,
                         "unit": "TFLOP/s", "frac": achieved_tf / peak_tf, "traffic": traffic,
                         "kernel": ("run_kernel_2d_p3 (one cooperative launch per timed segment: the sweeps, "
                                    "grid barriers and time control of all its steps)" if multi_step else
                                    f"sweep kernel d={d} n={p + 1} ({args.mode}: all sweep passes of the step)"),
                         "kernel_ms_per_step": kern_ms_per_step,
                         "kernel_share_of_step": share,
                         "kernel_timing": ("two CUDA events around the launch (= the timed segment)" if multi_step
                                           else "timed steps (two bracketing events per segment) x the sweep "
                                           "kernels' share of the step, measured in an instrumented replay of "
                                           "the same steps with CUDA events around every rerun / sweep launch"),
                         "flops_per_step_per_gpu": flops_total / K,
                         "peak_source": "profiles/fp64_peaks_r02.jsonl (measured DMMA m8n8k4; "
                                        f"DFMA {dfma} TF/s) — MEASURED_PEAKS.json has no fp64 entry",
                         "traffic_per_sweep_launch": traffic_launch,
                         "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one full sweep "
                                           "launch (profiles/r02/sweep_traffic.json) x sweep passes per timed step",
                         "hbm_alg_bytes_per_step": bytes_alg, "hbm_frac_of_measured": hbm_frac},
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    drv.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
