#!/bin/bash
# A/B variants of the product library for kernel experiments (not shipped):
#   tools/build_ab.sh name "-DFLAG=.. -DFLAG2" [name2 "flags2" ...]  -> tools/ab/lib_<name>.so
cd "$(dirname "$0")/.."
mkdir -p tools/ab
pids=()
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -shared $flags -o tools/ab/lib_$name.so paper_1801_08682_b200/csrc/aderdg_capi.cu > tools/ab/build_$name.log 2>&1 &
  pids+=($!)
done
rc=0
for p in "${pids[@]}"; do wait $p || rc=1; done
exit $rc
