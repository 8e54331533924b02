#!/bin/bash
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "c2 or c5 or union or ragged or edge or concurrent or bounds or maxh" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
: > gpurun_out/ab_${TAG}_summary.txt
for C in c2 c5; do for r in 1 2; do
  timeout 300 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}.log 2>&1
  echo "$C $(grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}.log)" >> gpurun_out/ab_${TAG}_summary.txt
done; done
