#!/bin/bash
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "c3 or wide or ragged or edge or bounds or host_pipeline or determinism" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
: > gpurun_out/ab_${TAG}_summary.txt
for r in 1 2 3; do for V in "X=1" "HOPF_TMG_BULK=0"; do
  timeout 300 env $V python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}.log 2>&1
  echo "$V $(grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}.log)" >> gpurun_out/ab_${TAG}_summary.txt
done; done
