#!/bin/bash
# dense kernel check: parity tests (dense only), then C4 bench (default kernel), short timeouts
TAG=${1:-d}
mkdir -p gpurun_out
timeout 150 python -m pytest tests -q -m gpu -k "dense or smoke" -x > gpurun_out/pytest_dense_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dense_$TAG.log
timeout 150 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4_$TAG.log
