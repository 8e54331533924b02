#!/bin/bash
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "distance or union or c5 or bounds" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
: > gpurun_out/ab_${TAG}_summary.txt
for V in "X=1" "HOPF_DIST_TMG=0"; do for r in 1 2; do
  timeout 300 env $V python bench.py --config c5d --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}.log 2>&1
  echo "$V $(grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}.log) $(grep -h -o '"kernel": "[^"]*"' gpurun_out/ab_${TAG}.log)" >> gpurun_out/ab_${TAG}_summary.txt
done; done
