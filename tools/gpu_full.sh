#!/bin/bash
# usage: tools/gpu_full.sh <tag> — full GPU test suite, smoke, default bench, launch lists (ncu)
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_$TAG.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default_$TAG.log
kill $SMI
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_$TAG.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_launch_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
CMD4="python bench.py --config c4 --M 200000 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD4 > gpurun_out/plain_launch4_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$TAG.csv $CMD4 > gpurun_out/ncu_launch4_$TAG.log 2>&1
echo done > gpurun_out/done_full_$TAG
