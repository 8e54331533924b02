#!/bin/bash
# usage: tools/gpu_bench_all.sh <tag>   (on the GPU box) — bench every config once
TAG=${1:-r01}
mkdir -p gpurun_out
for C in c3 c2 c5 c1 c4; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${C}_$TAG.log 2>&1
  echo "rc=$?" >> gpurun_out/bench_${C}_$TAG.log
done
