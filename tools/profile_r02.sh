#!/bin/bash
# ncu evidence of round 2 (run under gpurun, one GPU): per config the launch list of
# two steps (gpu__time_duration + DRAM bytes of every launch) -> gpurun_out/r02/launches_<cfg>.csv,
# and, for CONFIGS_FULL, one `--set full` capture of a sweep launch.  The report is exported
# on the box (raw page + SASS source page as gzipped CSV, read by tools/ncu_*.py through
# tools/_ncu_io.py) and deleted: gpurun_out/ travels back only below 64 MiB.
cd "$(dirname "$0")/.."
OUT=${OUT:-gpurun_out/r02}
mkdir -p $OUT
CONFIGS=${CONFIGS-"cfg2 cfg4 cfg3_p5 cfg3_p7 cfg3_p9 cfg1"}
CONFIGS_FULL=${CONFIGS_FULL-"cfg4"}
NCU=/usr/local/cuda/bin/ncu
for c in $CONFIGS; do
  python tools/prof_case.py $c 2 2 > $OUT/plain_$c.log 2>&1 && \
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
       --csv --log-file $OUT/launches_$c.csv python tools/prof_case.py $c 2 2 > $OUT/ncu_$c.log 2>&1
  echo "$c launches rc=$?"
done
for c in $CONFIGS_FULL; do
  python tools/prof_case.py $c 2 1 > $OUT/plain_full_$c.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:sweep_kernel -s 7 -c 1 \
       -f -o $OUT/full_$c python tools/prof_case.py $c 2 1 > $OUT/ncu_full_$c.log 2>&1
  echo "$c full rc=$?"
  if [ -f $OUT/full_$c.ncu-rep ]; then
    $NCU -i $OUT/full_$c.ncu-rep --page raw --csv | gzip > $OUT/full_${c}_raw.csv.gz
    $NCU -i $OUT/full_$c.ncu-rep --page source --csv --print-source sass | gzip > $OUT/full_${c}_sass.csv.gz
    $NCU -i $OUT/full_$c.ncu-rep --page details > $OUT/full_${c}_details.txt 2>&1
    rm -f $OUT/full_$c.ncu-rep
  fi
done
du -sh gpurun_out
