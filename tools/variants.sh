mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gpu_tests_v3.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_v3.log; tail -4 gpurun_out/gpu_tests_v3.log
ADG_KERNEL=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "p5 or p3" > gpurun_out/gpu_tests_k2.log 2>&1; echo k2rc=$?; tail -2 gpurun_out/gpu_tests_k2.log
for v in 1 2 3; do for c in cfg2 cfg3_p5; do
  st=17; [ $c = cfg3_p5 ] && st=7
  ADG_KERNEL=$v timeout 300 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_k$v.log 2>&1
  echo "$c k$v $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.3f'%d['ms_per_step'], '%.2f'%d['roofline']['achieved'], '%.3f'%d['roofline']['frac'], '%.2f'%d['config']['picard_mean'])" gpurun_out/bench_${c}_k$v.log 2>&1 | tail -1)"
done; done
