# tests + cfg2 / cfg3_p5 bench lines + ncu of the cfg2 sweep kernel (tag in $1)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gpu_tests_$1.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_$1.log; tail -3 gpurun_out/gpu_tests_$1.log
for c in ${CFGS:-cfg2 cfg3_p5}; do
  st=17; [ $c = cfg3_p5 ] && st=7
  timeout 300 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_$1.log 2>&1
  echo "$c $1 $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.3f'%d['ms_per_step'], '%.2f'%d['roofline']['achieved'], '%.3f'%d['roofline']['frac'], '%.2f'%d['config']['picard_mean'])" gpurun_out/bench_${c}_$1.log 2>&1 | tail -1)"
done
if [ "$2" = "ncu" ]; then
  timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 5 -c 1 -o gpurun_out/sweep_$1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$1.log 2>&1; echo ncu=$?
fi
