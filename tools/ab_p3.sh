# A/B of p=3 sweep-kernel variants on cfg2 (tag in $1, variants in $VARIANTS)
mkdir -p gpurun_out/abp3
for v in ${VARIANTS:-10 16 17}; do
  ADG_KERNEL=$v timeout 300 python bench.py --steps 17 --no-cpu-baseline --no-e2e > gpurun_out/abp3/cfg2_v${v}_$1.log 2>&1
  echo "cfg2 v$v $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.3e'%d['value'], '%.3f'%d['ms_per_step'], 'TF=%.2f'%d['roofline']['achieved'], '%.3f'%d['roofline']['frac'])" gpurun_out/abp3/cfg2_v${v}_$1.log 2>&1 | tail -1)"
done
