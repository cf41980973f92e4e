"""profiles/r02/sweep_traffic.json from the ncu launch lists of tools/profile_r02.sh.

    python tools/traffic_from_launches.py <dir with launches_<cfg>.csv> [profiled_steps=2]

tools/prof_case.py launches: priming sweep, finish, then per step rerun pass, sweep, finish
(stream launches, no graph).  The last 3 * profiled_steps launches are the profiled steps;
per step: DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and gpu__time_duration
of their sweep-kernel launches (the rerun pass exits early unless the step reruns)."""
import csv
import glob
import json
import os
import sys

src = sys.argv[1]
prof = int(sys.argv[2]) if len(sys.argv) > 2 else 2
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "second": 1.0}
out = {}
for path in sorted(glob.glob(os.path.join(src, "launches_*.csv"))):
    cfg = os.path.basename(path)[len("launches_"):-len(".csv")]
    with open(path) as fh:
        lines = fh.read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    launches = {}
    for r in rows:
        d = launches.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT[r["Metric Unit"]]
    # per step three launches (rerun pass, sweep, finish), or two where the sweep launch carries
    # the time control (2D p = 3: no finish_kernel after the priming step)
    tail = sorted(launches)[-3 * prof:]
    per_step = 3 if any("finish_kernel" in launches[i]["name"] for i in tail) else 2
    ids = sorted(launches)[-per_step * prof:]
    sweeps = [launches[i] for i in ids if "sweep_kernel" in launches[i]["name"]]
    allk = [launches[i] for i in ids]
    rd = sum(k.get("dram__bytes_read.sum", 0.0) for k in sweeps) / prof
    wr = sum(k.get("dram__bytes_write.sum", 0.0) for k in sweeps) / prof
    t_sweep = sum(k["gpu__time_duration.sum"] for k in sweeps) / prof
    t_all = sum(k["gpu__time_duration.sum"] for k in allk) / prof
    full = [k for k in sweeps if k["gpu__time_duration.sum"] > 0.2 * max(s["gpu__time_duration.sum"] for s in sweeps)]
    out[cfg] = {"kernel": sorted({k["name"].split("(")[0] for k in sweeps}),
                "dram_bytes_per_step": rd + wr, "dram_read": rd, "dram_write": wr,
                "sweep_ms_per_step_ncu": 1e3 * t_sweep, "all_kernels_ms_per_step_ncu": 1e3 * t_all,
                "sweep_share_of_step_ncu": t_sweep / t_all,
                "full_sweep_launches_per_step": len(full) / prof,
                "source": f"{path} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                          f"dram__bytes_write.sum --clock-control none; last {prof} steps of tools/prof_case.py)"}
json.dump(out, sys.stdout, indent=1)
print()
