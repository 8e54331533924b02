#!/bin/bash
# C2 kernel variants: parity subset, then bench with each env setting (3 runs each)
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "c2 or ragged or edge or determinism or concurrent or maxh" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
: > gpurun_out/ab_${TAG}_summary.txt
for V in "X=1" "$@"; do
  for r in 1 2 3; do
    timeout 300 env $V python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}.log 2>&1
    echo "$V $(grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}.log)" >> gpurun_out/ab_${TAG}_summary.txt
  done
done
