#!/bin/bash
# A/B: C3 with the TMEM kernel and the register kernel, alternating, 3 rounds each
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 200 python bench.py --config c3 --steps 50 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_tm_$i.log 2>&1
  HOPF_DIAG_TM=0 timeout 200 python bench.py --config c3 --steps 50 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_reg_$i.log 2>&1
done
