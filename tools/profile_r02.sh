#!/bin/bash
# ncu evidence of round 2 (run under gpurun, one GPU): per config the launch list of
# two steps (gpu__time_duration + DRAM bytes of every launch) -> profiles/r02/launches_<cfg>.csv,
# and, for CONFIGS_FULL, one `--set full` capture of a sweep launch -> gpurun_out/r02_<cfg>.ncu-rep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02
CONFIGS=${CONFIGS:-"cfg2 cfg4 cfg3_p5 cfg3_p7 cfg3_p9 cfg1"}
CONFIGS_FULL=${CONFIGS_FULL:-"cfg4"}
NCU=/usr/local/cuda/bin/ncu
for c in $CONFIGS; do
  python tools/prof_case.py $c 2 2 > gpurun_out/r02/plain_$c.log 2>&1 && \
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
       --csv --log-file gpurun_out/r02/launches_$c.csv python tools/prof_case.py $c 2 2 > gpurun_out/r02/ncu_$c.log 2>&1
  echo "$c launches rc=$?"
done
for c in $CONFIGS_FULL; do
  python tools/prof_case.py $c 2 1 > gpurun_out/r02/plain_full_$c.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:sweep_kernel -s 7 -c 1 \
       -o gpurun_out/r02/full_$c python tools/prof_case.py $c 2 1 > gpurun_out/r02/ncu_full_$c.log 2>&1
  echo "$c full rc=$?"
done
