"""Per-source-line shared-memory wavefronts of one kernel (run here, no GPU).
    python tools/ncu_smem_lines.py <report.ncu-rep> <mangled kernel name> [top]"""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.abspath(__file__)))
import _ncu_io
import csv, os, re, subprocess, sys, tempfile
from collections import defaultdict
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
lib = os.environ.get("ADG_PROFILE_LIB") or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1801_08682_b200", "libaderdg_b200.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if l.startswith(f".text.{kname}:"))
cur, a2l = None, {}
for l in dis[start + 1:]:
    if l.startswith(".text.") or l.strip().startswith(".section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        a2l[int(m.group(1), 16)] = cur
src = _ncu_io.page(rep, "sass")
rows = list(csv.reader(src.splitlines()))
h = rows[1]
ai, wf, wi, sa = h.index("Address"), h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal"), h.index("Source")
agg = defaultdict(lambda: [0, 0, set()])
tot = 0
base = int(rows[2][ai], 16)
for r in rows[2:]:
    try:
        a = int(r[ai], 16) - base; w = float(r[wf] or 0); wi_ = float(r[wi] or 0)
    except (ValueError, IndexError):
        continue
    if w == 0: continue
    k = a2l.get(a, ("?", 0))
    agg[k][0] += w; agg[k][1] += wi_; agg[k][2].add(r[sa].split()[0] if r[sa].split() else "")
    tot += w
print(f"total shared wavefronts {tot:.4g}")
for k, (w, wi_, ops) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]:24s} {k[1]:5d} {w:12.4g} {100*w/tot:5.1f}%  ideal {wi_:10.4g}  {sorted(ops)}")
