# full measurement pass: default bench line, reference arm, every BASELINE config on 1 GPU
mkdir -p gpurun_out/full
timeout 900 python bench.py > gpurun_out/full/bench_default.json 2> gpurun_out/full/bench_default.err; echo "default rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/full/bench_reference.json 2> gpurun_out/full/bench_reference.err; echo "reference rc=$?"
timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/full/bench_cfg1.json 2>&1; echo "cfg1 rc=$?"
timeout 600 python bench.py --config cfg3_p5 --steps 7 --no-cpu-baseline > gpurun_out/full/bench_cfg3_p5.json 2>&1; echo "p5 rc=$?"
timeout 600 python bench.py --config cfg3_p7 --steps 3 --no-cpu-baseline > gpurun_out/full/bench_cfg3_p7.json 2>&1; echo "p7 rc=$?"
timeout 600 python bench.py --config cfg3_p9 --steps 1 --no-cpu-baseline > gpurun_out/full/bench_cfg3_p9.json 2>&1; echo "p9 rc=$?"
timeout 900 python bench.py --config cfg4 --steps 7 --no-cpu-baseline --no-e2e > gpurun_out/full/bench_cfg4.json 2>&1; echo "cfg4 rc=$?"
timeout 1200 python bench.py --config cfg5_1gpu --steps 2 --no-cpu-baseline --no-e2e > gpurun_out/full/bench_cfg5_1gpu.json 2>&1; echo "cfg5 rc=$?"
for f in gpurun_out/full/*.json; do python -c "
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
  r=d.get('roofline') or {}
  e=d.get('e2e') or {}
  c=d.get('cpu_baseline') or {}
  print(sys.argv[1].split('/')[-1], '%.3e'%d['value'], 'ms=%.3f'%d['ms_per_step'], 'TF=%.2f'%r.get('achieved',0), 'frac=%.3f'%r.get('frac',0), 'e2e=%.3e'%e.get('value',0), 'cpu=%.3e'%c.get('value',0), d.get('clocks'))
except Exception as ex: print(sys.argv[1], 'ERR', ex)
" $f; done
