#!/usr/bin/env python
"""bench.py — fp64 DoF-updates/s of the fused ADER-DG Euler step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

Metric (BASELINE.json): fp64 DoF-updates/s for 3D Euler ADER-DG at order p,
DoF = cells * (p+1)^d * m.  Default workload = BASELINE config 2 (3D, p=3,
27^3 periodic cells, Gaussian bump + seeded 1e-3 density noise, Rusanov,
CFL 0.9/(d(2p+1)), c_dt 0.99): a "step" is one fused realisation step of
the whole grid (rerun pass when the optimistic step fails, fused
Riemann/corrector/update/CFL/predictor sweep, device time control).
N > 1: x-slab decomposition, one process per GPU (torchrun), NCCL halo
exchange + lambda all-reduce per step; total work fixed (strong scaling).

Reported on one JSON line (rank 0):
  value      DoF-updates/s, device-timed (CUDA events, max over ranks), state resident in HBM
  e2e        same metric through the C ABI with host buffers: per step H2D of Q from
             pinned memory, adg step, D2H of Q (wall clock, max over ranks)
  roofline   dominant kernel (sweep_kernel: fused sweep + rerun passes), algorithmic
             flops (paper_1801_08682_b200/roofline.py, measured Picard counts) / its
             CUDA-event time, against the measured FP64 peak (profiles/fp64_peaks_r01.jsonl)
  cpu_baseline  the CPU oracle port (oracle/aderdg_oracle.py, batched numpy) timed on
             this host on a bounded sample (rank 0, N=1 only)
--impl reference: times the oracle port (the reference is CPU-only Python; the oracle is
its batched restatement) on a bounded sample of the same workload, rank 0 only.
"""

import argparse
import ctypes
import json
import os
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
    "cfg5_1gpu": dict(d=3, L=4, p=9, scenario="fourier", steps=5,
                      desc="BASELINE cfg5: 3D Euler p=9, 81^3 periodic, random Fourier state, 5 steps"),
    # 81^3 p=5 with the specified noise aborts at step 10 (NumericalError, cell 208997; measured
    # on the GPU path): timed on the 9 steps before the abort
    "cfg4": dict(d=3, L=4, p=5, scenario="bump", steps=9,
                 desc="BASELINE cfg4: 3D Euler p=5, 81^3 periodic, bump+1e-3 noise (9 pre-abort steps)"),
}

PEAKS_FILE = os.path.join(REPO, "profiles", "fp64_peaks_r01.jsonl")
NCU_TRAFFIC_FILE = os.path.join(REPO, "profiles", "sweep_traffic_r01.json")


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


def cpu_oracle_rate(cfgd, steps, warmup, L_override=None):
    """Time the CPU oracle (oracle/aderdg_oracle.py) on a bounded sample, in
    episodes of at most the configured step count (restarts untimed)."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import aderdg_oracle as O
    from paper_1801_08682_b200 import roofline, scenarios
    d, p = cfgd["d"], cfgd["p"]
    L = L_override or cfgd["L"]
    E = cfgd["steps"]
    Q0 = scenarios.build(cfgd["scenario"], d, L, p)
    times, first = [], True
    while len(times) < steps:
        drv = O.FusedDriver(Q0.copy(), d, p, L)
        warm = max(1, warmup) if first else 1   # the first step carries the priming sweep
        for _ in range(warm):
            drv.step()
        for _ in range(min(steps - len(times), max(1, E - warm))):
            t0 = time.perf_counter()
            drv.step()
            times.append(time.perf_counter() - t0)
        first = False
    dofs = roofline.dof(d, p, 3 ** (d * L))
    try:
        from threadpoolctl import threadpool_info
        blas = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        blas = 1
    return dofs * len(times) / sum(times), times, blas, L


def run_reference(args, cfgd):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # bounded sample: same d, p and state family on the 9^3 (3D) / 27^2 (2D) grid
    L_s = 2 if cfgd["d"] == 3 else 3
    rate, times, blas, L = cpu_oracle_rate(cfgd, args.steps, args.warmup, L_override=L_s)
    sample = (f"oracle port (batched numpy restatement of the reference fused driver), "
              f"{3 ** L}^{cfgd['d']} cells p={cfgd['p']}, {len(times)} steps after priming+"
              f"{args.warmup} warm-up; BLAS threads {blas}, numpy elementwise single-threaded")
    ms = 1e3 * sum(times) / len(times)
    line = {
        "impl": "reference", "metric": "fp64 DoF-updates/s (3D Euler ADER-DG, fused step)",
        "value": rate, "unit": "DoF-updates/s", "n_gpus": args.gpus, "steps": len(times),
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfgd["desc"], "d": cfgd["d"], "p": cfgd["p"],
                   "cells_sample": 3 ** (cfgd["d"] * L)},
        "cpu_baseline": {"value": rate, "unit": "DoF-updates/s", "cores": blas, "kind": "port",
                         "sample": sample},
        "e2e": {"value": rate, "unit": "DoF-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=17)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="fused", choices=["fused", "straightforward"],
                    help="driver: fused single-touch (north star) or the straightforward passes")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfgd = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfgd)

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
    if staged:
        local = 0
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
    # N > 1: the timed steps are enqueued from C over the library's own NCCL
    # communicator (adg_run_timed_mgpu); ADG_MGPU_PY=1 keeps the per-step Python loop
    native = world > 1 and not staged and os.environ.get("ADG_MGPU_PY") != "1"
    if native:
        try:
            drv.init_native_comm()
        except RuntimeError as e:        # same verdict on every rank (parallel.SlabDriver)
            print(f"[bench] native NCCL step loop unavailable ({e}); per-step Python loop", file=sys.stderr)
            native = False
    K = args.steps
    clocks = ClockSampler(local)
    seg_ms, kern_ms, recs, launches = [], 0.0, [], 0
    remaining, first = K, True
    clocks_started = False
    while remaining > 0:
        if not first:
            drv.load(Q0)
        warm = args.warmup if first else 1
        for _ in range(warm):
            drv.enqueue_step()
        h.call("adg_sync")
        step0 = h.lib.adg_step_count(h.h)
        n = min(remaining, max(1, E - warm))
        if world == 1:
            # single GPU: the C side enqueues the n steps back to back (one CUDA graph)
            # with CUDA events around the segment only; the per-launch kernel events
            # cost graph-node gaps, so the kernel time comes from a replay (below)
            torch.cuda.synchronize()
            if not clocks_started:
                clocks.start()
                clocks_started = True
                time.sleep(0.05)
            tout = (ctypes.c_double * 2)()
            h.call("adg_run_timed_ex", n, 0, tout)
            seg_ms.append(tout[0])
        elif native:
            barrier()
            torch.cuda.synchronize()
            if not clocks_started:
                clocks.start()
                clocks_started = True
                time.sleep(0.05)
            seg, _ = drv.run_timed(n, flags=0)
            barrier()
            seg_ms.append(seg)
        else:
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n)]
            start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            torch.cuda.synchronize()
            if not clocks_started:
                clocks.start()
                clocks_started = True
                time.sleep(0.05)
            start.record()
            for i in range(n):
                # rerun -> { halo exchange (NCCL stream) || interior planes } -> boundary
                # planes -> all-reduce -> time control (parallel.SlabDriver.enqueue_step)
                e0, e1, e2, e3 = ev[i]
                e0.record()
                h.call("adg_phase_rerun")
                e1.record()
                pending = drv.halo.start(drv.tr[h.lib.adg_trace_parity(h.h)])
                e2.record()
                h.call("adg_phase_sweep_part", _lib.ADG_PART_INTERIOR)
                drv.halo.wait(pending)
                h.call("adg_phase_sweep_part", _lib.ADG_PART_BOUNDARY)
                e3.record()
                drv.halo.reduce(drv.red)
                h.call("adg_phase_finish")
            stop.record()
            torch.cuda.synchronize()
            barrier()
            h.call("adg_sync")
            seg_ms.append(start.elapsed_time(stop))
            kern_ms += sum(e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3]) for e in ev)
        seg_recs = h.step_records(step0 + 1, n)
        recs += seg_recs
        graph_steps = world == 1 or (native and os.environ.get("ADG_MGPU_NO_GRAPH") is None)
        if graph_steps and os.environ.get("ADG_NO_COND_RERUN") is None:
            # graph steps: sweep + finish, and the rerun pass only where its conditional
            # node fires (the segment's first step, whose condition defaults to 1, and steps
            # after a finish that asked for a rerun)
            launches += 2 * n + 1 + sum(1 for r in seg_recs[1:] if r.reruns)
        else:
            launches += 3 * n     # rerun-pass sweep_kernel + sweep_kernel + finish_kernel
        remaining -= n
        first = False
    clk = clocks.stop()
    kern_seg_ms, replay_recs = sum(seg_ms), []
    if world == 1 or native:
        # instrumented replay of the timed segments (same initial states, same launch
        # sequence): CUDA events around every rerun / sweep launch give the kernel time
        kern_ms, kern_seg_ms, remaining, firstr = 0.0, 0.0, K, True
        while remaining > 0:
            drv.load(Q0)
            warm = args.warmup if firstr else 1
            for _ in range(warm):
                drv.enqueue_step()
            h.call("adg_sync")
            n = min(remaining, max(1, E - warm))
            tout = (ctypes.c_double * 2)()
            s0 = h.lib.adg_step_count(h.h)
            if world == 1:
                h.call("adg_run_timed_ex", n, _lib.ADG_TIMED_KERNEL_EVENTS, tout)
            else:
                barrier()
                tout[0], tout[1] = drv.run_timed(n, flags=_lib.ADG_TIMED_KERNEL_EVENTS)
                barrier()
            kern_ms += tout[1]
            kern_seg_ms += tout[0]
            rr = h.step_records(s0 + 1, n)
            replay_recs += rr
            if os.environ.get("ADG_BENCH_DEBUG"):
                print("[replay] seg %.3f kern %.3f reruns %d iters %d preds %d | timed: seg %s iters %d preds %d" % (
                    tout[0], tout[1], sum(r.reruns for r in rr), sum(r.picard_iters for r in rr),
                    sum(r.predicts for r in rr), seg_ms, sum(r.picard_iters for r in recs),
                    sum(r.predicts for r in recs)), file=sys.stderr)
            remaining -= n
            firstr = False
    elapsed_ms = max_over_ranks(sum(seg_ms))
    iters = sum(r.picard_iters for r in recs)
    preds = sum(r.predicts for r in recs)
    reruns = sum(r.reruns for r in recs)
    local_cells = drv.n_local
    flops = roofline.flops_step(d, p, local_cells, iters, preds)
    ms_per_step = elapsed_ms / K
    value = dofs * K / (elapsed_ms * 1e-3)
    kern_ms_per_step = kern_ms / K
    achieved_tf = flops / (kern_ms * 1e-3) / 1e12
    dfma, dmma, hbm = load_peaks()
    peak_tf = dmma or dfma or 37.1
    traffic = None
    try:
        with open(NCU_TRAFFIC_FILE) as fh:
            tinfo = json.load(fh)
        traffic = tinfo.get(args.config, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
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
                        "up to 16 wave-aligned cell chunks" if world == 1 else
                        "adg_load_state (pinned H2D) + phase step + adg_store_state (D2H), per step")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        L_s = 2 if d == 3 else L
        rate, times, blas, Ls = cpu_oracle_rate(cfgd, 2, 0, L_override=L_s)
        cpu = {"value": rate, "unit": "DoF-updates/s", "cores": blas, "kind": "port",
               "sample": (f"oracle/aderdg_oracle.py (batched numpy restatement of the reference "
                          f"fused driver), {3 ** Ls}^{d} cells p={p}, 2 steps after priming; "
                          f"BLAS threads {blas}, numpy elementwise single-threaded")}

    if rank == 0:
        line = {
            "metric": "fp64 DoF-updates/s (3D Euler ADER-DG, fused step)",
            "value": value, "unit": "DoF-updates/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfgd["desc"], "d": d, "p": p, "L": L, "cells": cells,
                       "driver": args.mode,
                       "nodes": cells * (p + 1) ** d, "dof": dofs,
                       "parallelism": f"x-slab x{world}" if world > 1 else "single GPU",
                       "exchange": (None if world == 1 else "gloo staged (functional only)" if staged
                                    else "library NCCL comm, steps enqueued from C" if native
                                    else "torch.distributed NCCL, per-step Python loop"),
                       "l2": "no flush: per-step working set (Q,D r/w + 2 trace parities) "
                             f"{roofline.bytes_step(d, p, cells) / 1e6:.0f} MB > 126 MB L2",
                       "episode_steps": E, "episodes": len(seg_ms),
                       "reruns_in_timed": reruns, "picard_mean": iters / max(preds, 1)},
            # compute-bound on the FP64 datapath; the peak is the measured FP64 tensor-core
            # (DMMA) throughput, which the CUDA-core DFMA pipe shares (contract: hbm | tensor)
            "roofline": {"bound": "tensor", "datapath": "fp64 (DMMA m8n8k4 + DFMA)",
                         "achieved": achieved_tf, "peak": peak_tf,
                         "unit": "TFLOP/s", "frac": achieved_tf / peak_tf, "traffic": traffic,
                         "kernel": f"sweep kernel d={d} n={p + 1} ({args.mode}: all sweep passes of the step)",
                         "kernel_ms_per_step": kern_ms_per_step,
                         "kernel_share_of_step": kern_ms / kern_seg_ms,
                         "kernel_timing": ("CUDA events around every rerun / sweep launch in an "
                                           "instrumented replay of the timed steps (same states and "
                                           "launches); the timed graph carries only its two bracketing "
                                           "events" if (world == 1 or native) else
                                           "CUDA events around every sweep launch in the timed steps"),
                         "flops_per_step_per_gpu": flops / K if K else 0,
                         "peak_source": "profiles/fp64_peaks_r01.jsonl (measured DMMA m8n8k4; "
                                        f"DFMA {dfma} TF/s) — MEASURED_PEAKS.json has no fp64 entry",
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
