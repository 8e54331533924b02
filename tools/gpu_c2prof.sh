#!/bin/bash
# C2: parity subset, bench (3 runs), one ncu --set full capture of the tmg kernel
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "c2 or ragged or edge or determinism or concurrent or maxh" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
: > gpurun_out/ab_${TAG}_summary.txt
for r in 1 2 3; do
  timeout 300 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}.log 2>&1
  echo "$(grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}.log)" >> gpurun_out/ab_${TAG}_summary.txt
done
bash tools/gpu_ncu_src.sh $TAG c2 1000000 hopf_diag_tmg
