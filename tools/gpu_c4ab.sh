#!/bin/bash
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "dense or c4 or bounds or concurrent" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
: > gpurun_out/ab_${TAG}_summary.txt
for r in 1 2; do
  timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}.log 2>&1
  echo "$(grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}.log) $(grep -h -o '"sm_mhz": [0-9.]*' gpurun_out/ab_${TAG}.log)" >> gpurun_out/ab_${TAG}_summary.txt
done
