#!/bin/bash
# paper-protocol context lines (Tables 1 and 4 setup): p<n>_<id|diag>_<l1|l2>, M = 1e6
TAG=${1:-r02}
mkdir -p gpurun_out
: > gpurun_out/pprot_$TAG.jsonl
for N in 4 8 12 16; do for J in id diag; do for H in l1 l2; do
  timeout 300 python bench.py --config p${N}_${J}_${H} --steps 20 --warmup 3 --no-e2e 2>gpurun_out/pprot_err.log | grep '^{' >> gpurun_out/pprot_$TAG.jsonl
done; done; done
