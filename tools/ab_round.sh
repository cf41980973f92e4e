# session-3 A/B: BLK p=5 mapping (31) and TMEM divergence history at p=9 (42)
ADG_KERNEL=31 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t31.log 2>&1; echo "t31 rc=$?"
ADG_KERNEL=42 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t42.log 2>&1; echo "t42 rc=$?"
bash tools/ab5.sh "3 31"
for v in 41 40 42; do
  ADG_KERNEL=$v timeout 300 python bench.py --config cfg3_p9 --steps 1 --no-cpu-baseline --no-e2e > gpurun_out/abp9_k$v.log 2>&1
  echo "p9 k$v $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.3f'%d['ms_per_step'], '%.2f'%d['roofline']['achieved'], '%.3f'%d['roofline']['frac'])" gpurun_out/abp9_k$v.log 2>&1 | tail -1)"
done
