#!/bin/bash
# usage: tools/gpu_cycle.sh <tag> [ncu configs...]  — pytest -m gpu, bench all configs, ncu full on listed configs
TAG=${1:-r01}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
bash tools/gpu_bench_all.sh $TAG
for CFG in "$@"; do
  CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  timeout 300 $CMD > gpurun_out/plain_${CFG}_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:hopf -s 3 -c 1 -o gpurun_out/prof_${CFG}_$TAG $CMD > gpurun_out/ncu_full_${CFG}_$TAG.log 2>&1
done
echo done > gpurun_out/done_$TAG
