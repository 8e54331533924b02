#!/bin/bash
TAG=${1:-tm}
mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -k "not dense" -x > gpurun_out/pytest_tm_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tm_$TAG.log
timeout 200 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_$TAG.log 2>&1
HOPF_DIAG_TM=0 timeout 200 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_reg_$TAG.log 2>&1
