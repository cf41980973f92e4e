# ncu evidence for the current default kernels (tag in $1): launch list of the
# cfg2 bench and one --set full capture of the sweep kernel per config
mkdir -p gpurun_out/prof_$1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_$1/plain.log 2>&1; echo plain=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof_$1/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_$1/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 5 -c 1 -o gpurun_out/prof_$1/sweep_cfg2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_$1/ncu_cfg2.log 2>&1; echo full_cfg2=$?
for c in ${CFGS:-cfg3_p5}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 -o gpurun_out/prof_$1/sweep_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_$1/ncu_$c.log 2>&1; echo full_$c=$?
done
