#!/bin/bash
# usage: tools/gpu_buildab.sh <tag> <config> "<flags A>" "<flags B>" ...: rebuild the library with
# each set of extra nvcc flags (HOPF_EXTRA_NVCC_FLAGS) and bench the config 3 times per build
TAG=$1; CFG=$2; shift 2
mkdir -p gpurun_out
: > gpurun_out/bab_${TAG}_summary.txt
for F in "$@"; do
  HOPF_EXTRA_NVCC_FLAGS="$F" python -m paper_1605_01799_b200.build --force > gpurun_out/bab_${TAG}_build.log 2>&1 || { echo "build failed: $F" >> gpurun_out/bab_${TAG}_summary.txt; continue; }
  for r in 1 2 3; do
    timeout 300 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bab_${TAG}.log 2>&1
    echo "[$F] $(grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/bab_${TAG}.log)" >> gpurun_out/bab_${TAG}_summary.txt
  done
done
