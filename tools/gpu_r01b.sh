#!/bin/bash
# session-3 check: full GPU tests, dense v3 vs v2 bench, default bench
TAG=${1:-r01b}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_tc2_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4_tc2_$TAG.log
HOPF_DENSE_KERNEL=tc1 timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_tc1_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4_tc1_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_default_$TAG.log
echo done > gpurun_out/done_$TAG
