# full measurement pass (run under gpurun, one GPU): the default bench line, the reference arm,
# every BASELINE config on one GPU -> gpurun_out/full/
mkdir -p gpurun_out/full
timeout 900 python bench.py > gpurun_out/full/bench_default.json 2> gpurun_out/full/bench_default.err; echo "default rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/full/bench_reference.json 2> gpurun_out/full/bench_reference.err; echo "reference rc=$?"
for c in cfg1 cfg2 cfg3_p5 cfg3_p7 cfg3_p9; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/full/bench_$c.json 2> gpurun_out/full/bench_$c.err; echo "$c rc=$?"
done
timeout 1200 python bench.py --config cfg5 --no-cpu-baseline --no-e2e > gpurun_out/full/bench_cfg5_1gpu.json 2> gpurun_out/full/bench_cfg5_1gpu.err; echo "cfg5 rc=$?"
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
