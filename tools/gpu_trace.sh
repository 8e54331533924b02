#!/bin/bash
mkdir -p gpurun_out
HOPF_TC3_TRACE=gpurun_out/tc3_trace.txt timeout 300 python bench.py --config c4 --M 400000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/trace_bench.log 2>&1
echo rc=$? >> gpurun_out/trace_bench.log
