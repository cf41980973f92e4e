# A/B of the high-order kernel variants on cfg3 p=7 / p=9 (variant list in $1)
for v in $1; do
  for c in cfg3_p7 cfg3_p9; do
    st=3; [ $c = cfg3_p9 ] && st=1
    ADG_KERNEL=$v timeout 300 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e > gpurun_out/abho_${c}_k$v.log 2>&1
    echo "$c k$v $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.3f'%d['ms_per_step'], '%.2f'%d['roofline']['achieved'], '%.3f'%d['roofline']['frac'])" gpurun_out/abho_${c}_k$v.log 2>&1 | tail -1)"
  done
done
