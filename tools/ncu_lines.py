"""Attribute ncu warp-stall samples of one kernel to CUDA source lines (run here, no GPU).

    python tools/ncu_lines.py <report.ncu-rep> <mangled kernel name> [top]

Maps SASS addresses of the ncu source page onto `nvdisasm -g` line info of the
in-tree library's cubin (the report must come from the same build)."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.abspath(__file__)))
import _ncu_io
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
lib = os.environ.get("ADG_PROFILE_LIB") or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1801_08682_b200", "libaderdg_b200.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
lines = dis.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{kname}:"))
cur, a2l = None, {}
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.strip().startswith(".section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        a2l[int(m.group(1), 16)] = cur
src = _ncu_io.page(rep, "sass")
rows = list(csv.reader(src.splitlines()))
h = rows[1]
ai, ws, ie = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = rows[2:]
f = lambda x: float(x) if x not in ("", "-") else 0.0
base = int(data[0][ai], 16)
agg = defaultdict(lambda: [0.0, 0.0])
tot = sum(f(r[ws]) for r in data)
for r in data:
    k = a2l.get(int(r[ai], 16) - base, ("?", 0))
    agg[k][0] += f(r[ws])
    agg[k][1] += f(r[ie])
srcs = {}
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    text = ""
    for d in ("paper_1801_08682_b200/csrc",):
        p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), d, k[0])
        if os.path.exists(p):
            srcs.setdefault(p, open(p).read().splitlines())
            text = srcs[p][k[1] - 1].strip() if k[1] - 1 < len(srcs[p]) else ""
    print(f"{k[0][:22]:22s} {k[1]:5d} {v[0] / tot * 100:5.1f}%  inst={v[1]:12.0f}  {text[:70]}")
