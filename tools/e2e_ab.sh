# A/B of the pipelined host step (adg_step_host): chunk schedules
mkdir -p gpurun_out/e2e
run() { # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline > gpurun_out/e2e/$tag.json 2> gpurun_out/e2e/$tag.err
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], 'value %.4e'%d['value'], 'e2e %.4e'%d['e2e']['value'], 'e2e_ms %.3f'%d['e2e']['ms_per_step'])" gpurun_out/e2e/$tag.json $tag
}
run c16 ADG_HOST_SWEEP_STREAMS=1
run c12 ADG_HOST_SWEEP_STREAMS=1 ADG_HOST_CHUNKS=12
run w1 ADG_HOST_SWEEP_STREAMS=1 ADG_HOST_WAVES=1,2,4,4,4,4,2,1,1
run w2 ADG_HOST_SWEEP_STREAMS=1 ADG_HOST_WAVES=1,1,2,3,3,3,3,3,2,1,1
run w3 ADG_HOST_SWEEP_STREAMS=1 ADG_HOST_WAVES=1,2,3,5,5,3,2,1,1
run w4 ADG_HOST_SWEEP_STREAMS=1 ADG_HOST_WAVES=1,1,2,2,2,2,2,2,2,2,2,1,1,1
run w5 ADG_HOST_SWEEP_STREAMS=4 ADG_HOST_WAVES=1,1,2,3,3,3,3,3,2,1,1
run w6 ADG_HOST_SWEEP_STREAMS=1 ADG_HOST_WAVES=2,3,4,4,4,3,2,1
ADG_HOST_SWEEP_STREAMS=1 ADG_HOST_WAVES=1,1,2,3,3,3,3,3,2,1,1 ADG_HOST_TRACE=1 timeout 300 python bench.py --no-cpu-baseline --steps 3 > /dev/null 2> gpurun_out/e2e/trace_w2.err
