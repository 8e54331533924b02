#!/bin/bash
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "ell or linf or maxh or ragged or bounds" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
: > gpurun_out/ab_${TAG}_summary.txt
for C in c2e c2i c2h; do for V in "X=1" "HOPF_DIAG_TMG=0"; do
  timeout 300 env $V python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}.log 2>&1
  echo "$C $V $(grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}.log) $(grep -h -o '"kernel": "[^"]*"' gpurun_out/ab_${TAG}.log)" >> gpurun_out/ab_${TAG}_summary.txt
done; done
