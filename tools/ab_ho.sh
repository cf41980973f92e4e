# A/B of the high-order kernel variants: parity on p >= 6 cases + cfg3 p7/p9 bench lines
mkdir -p gpurun_out/abho
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "p7 or p9 or 6-3 or 7-3 or 8-2 or 9-2 or p6" > gpurun_out/abho/par_$1.log 2>&1; echo "parity rc=$? $(tail -1 gpurun_out/abho/par_$1.log)"
for v in ${VARIANTS:-3 15}; do
  for c in cfg3_p7 cfg3_p9; do
    st=3; [ $c = cfg3_p9 ] && st=1
    ADG_KERNEL=$v timeout 600 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e > gpurun_out/abho/${c}_v$v.log 2>&1
    echo "$c v$v $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.3f'%d['ms_per_step'], 'TF=%.2f'%d['roofline']['achieved'], '%.3f'%d['roofline']['frac'])" gpurun_out/abho/${c}_v$v.log 2>&1 | tail -1)"
  done
done
