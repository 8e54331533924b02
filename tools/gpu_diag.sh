#!/bin/bash
# diag/union check: parity tests (diag, union, edge cases), then C3 / C2 / C5 benches
TAG=${1:-d}
mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -k "not dense" -x > gpurun_out/pytest_diag_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_diag_$TAG.log
for C in c3 c2 c5; do
  timeout 200 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${C}_$TAG.log
done
