mkdir -p gpurun_out/ev
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "run_timed or step_host" > gpurun_out/ev/tests.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/ev/tests.log
for c in cfg1 cfg2; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/ev/$c.json 2>gpurun_out/ev/$c.err
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
print(sys.argv[2], 'ms %.4f'%d['ms_per_step'], 'value %.4e'%d['value'], 'TF %.2f'%r['achieved'], 'share %.3f'%r['kernel_share_of_step'], 'e2e %.3e'%d['e2e']['value'])" gpurun_out/ev/$c.json $c
done
