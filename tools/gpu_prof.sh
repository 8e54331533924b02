#!/bin/bash
# usage: tools/gpu_prof.sh <tag> [config]   (on the GPU box) — pytest, bench, ncu launch list + full capture
TAG=${1:-r01}; CFG=${2:-c3}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --config $CFG --steps 100 --warmup 5 > gpurun_out/bench_${CFG}_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${CFG}_$TAG.log
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hopf -s 3 -c 1 -o gpurun_out/prof_${CFG}_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "done" >> gpurun_out/ncu_full_$TAG.log
