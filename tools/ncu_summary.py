"""Summarise an ncu --set full report of the sweep kernel (run here, no GPU):
    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--sass]"""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.abspath(__file__)))
import _ncu_io
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = _ncu_io.page(rep, "raw")
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size", "launch__block_size"]
out = {}
for i, name in enumerate(h):
    if name in want:
        out[name] = (v[i], u[i])
for k in want:
    if k in out:
        print(f"{k:80s} {out[k][0]} {out[k][1]}")
items = []
for i, name in enumerate(h):
    if "smsp__average_warps_issue_stalled" in name and name.endswith("per_issue_active.ratio"):
        try:
            items.append((float(v[i]), name.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("stalls (cycles per issued instruction):", ", ".join(f"{n}={x:.2f}" for x, n in sorted(items, reverse=True)[:9]))
if "--sass" in sys.argv:
    src = _ncu_io.page(rep, "sass")
    rows = list(csv.reader(src.splitlines()))
    hh = rows[1]
    si, ie = hh.index("Source"), hh.index("Instructions Executed")
    ws = hh.index("Warp Stall Sampling (All Samples)")
    cnt, stall = Counter(), Counter()
    for row in rows[2:]:
        toks = row[si].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        cnt[op] += float(row[ie] or 0)
        stall[op] += float(row[ws] or 0)
    tot = sum(cnt.values())
    tots = sum(stall.values())
    print("instruction mix (executed warp-instructions):")
    for op, c in cnt.most_common(18):
        print(f"  {op:10s} {c / tot * 100:5.1f}%   stall-samples {stall[op] / tots * 100:5.1f}%")
