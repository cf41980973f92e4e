#!/bin/bash
# compute-sanitizer over every product kernel path (tools/sanitize_case.py);
# logs under profiles/r02/sanitizer/<tool>_<case>.log, summary in summary.txt
cd "$(dirname "$0")/.."
OUT=profiles/r02/sanitizer
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
CASES=${CASES:-"p3 p5 p7 p9 gen2d p4 sf adv lim host stream"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck initcheck"}
: > $OUT/summary.txt
for tool in $TOOLS; do
  for c in $CASES; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check full"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
    timeout 900 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_case.py $c > $OUT/${tool}_${c}.log 2>&1
    rc=$?
    s=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY" $OUT/${tool}_${c}.log | tr '\n' ' ')
    echo "$tool $c rc=$rc $s" | tee -a $OUT/summary.txt
  done
done
