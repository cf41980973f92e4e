"""Run a few realisation steps in one driver mode (for ncu DRAM-traffic capture).

    python tools/traffic_ratio.py --mode fused|straightforward [--config cfg2] [--steps 2] [--warmup 3]

Under `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--csv --log-file X` the last 3*steps launches are the measured steps (3 launches per
step in both modes); `tools/traffic_ratio.py --parse fused.csv straightforward.csv`
prints bytes per step and the fused / straightforward ratio (the paper's
single-touch claim, Table 1 / SPEC traffic model)."""
import argparse
import csv
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def run(args):
    import torch
    sys.path.insert(0, REPO)
    from bench import CONFIGS
    from paper_1801_08682_b200 import scenarios
    from paper_1801_08682_b200.parallel import SlabDriver
    c = CONFIGS[args.config]
    Q0 = scenarios.build(c["scenario"], c["d"], c["L"], c["p"])
    torch.cuda.set_device(0)
    drv = SlabDriver(Q0, c["d"], c["L"], c["p"], 0, 1, 0, mode=args.mode,
                     forced_dt=args.forced_dt)
    for _ in range(args.warmup + args.steps):
        drv.enqueue_step()
    drv.handle.call("adg_sync")
    print(json.dumps({"mode": args.mode, "steps": drv.handle.lib.adg_step_count(drv.handle.h)}))


def parse(paths):
    out = {}
    for p in paths:
        rows = list(csv.reader(open(p)))
        hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
        h = rows[hdr]
        idc, kn, mn, mv, mu = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
        launches = {}
        for r in rows[hdr + 1:]:
            if len(r) <= mv:
                continue
            d = launches.setdefault(int(r[idc]), {"kernel": r[kn]})
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                     "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(r[mu], 1)
            d[r[mn]] = float(r[mv].replace(",", "")) * scale
        ids = sorted(launches)
        mode = "straightforward" if "straight" in os.path.basename(p) else "fused"
        steps = int(os.environ.get("STEPS", "2"))
        last = [launches[i] for i in ids[-3 * steps:]]
        byt = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in last) / steps
        tim = sum(x.get("gpu__time_duration.sum", 0) for x in last) / steps
        out[mode] = {"dram_bytes_per_step": byt, "kernel_time_per_step_s": tim,
                     "launches": [x["kernel"][:40] for x in last[:3]]}
    if "fused" in out and "straightforward" in out:
        out["ratio_fused_over_straightforward"] = (out["fused"]["dram_bytes_per_step"] /
                                                   out["straightforward"]["dram_bytes_per_step"])
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if "--parse" in sys.argv:
        parse([a for a in sys.argv[1:] if a != "--parse"])
    else:
        ap = argparse.ArgumentParser()
        ap.add_argument("--mode", default="fused")
        ap.add_argument("--config", default="cfg2")
        ap.add_argument("--steps", type=int, default=2)
        ap.add_argument("--warmup", type=int, default=3)
        ap.add_argument("--forced-dt", type=float, default=None)
        run(ap.parse_args())
