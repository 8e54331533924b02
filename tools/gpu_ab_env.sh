#!/bin/bash
# usage: tools/gpu_ab_env.sh <tag> <config> <ENV=VAL for B> [pytest -k expr]
# A/B of one config: A = default build, B = with the env var set; 3 alternating runs each
TAG=$1; CFG=$2; ENVB=$3; KEXPR=$4
mkdir -p gpurun_out
if [ -n "$KEXPR" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x -k "$KEXPR" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
fi
for r in 1 2 3; do
  timeout 300 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}_A$r.log 2>&1
  timeout 300 env $ENVB python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}_B$r.log 2>&1
done
grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}_A*.log > gpurun_out/ab_${TAG}_summary.txt
echo B >> gpurun_out/ab_${TAG}_summary.txt
grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}_B*.log >> gpurun_out/ab_${TAG}_summary.txt
