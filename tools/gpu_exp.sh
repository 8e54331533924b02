#!/bin/bash
# trace experiments with alternative builds of libhopf.so placed under exp/
mkdir -p gpurun_out
cp paper_1605_01799_b200/libhopf.so /tmp/libhopf_orig.so
for L in exp/libhopf_*.so; do
  T=$(basename $L .so)
  cp $L paper_1605_01799_b200/libhopf.so
  HOPF_TC3_TRACE=gpurun_out/trace_$T.txt timeout 120 python bench.py --config c4 --M 400000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/exp_$T.log 2>&1
  echo rc=$? >> gpurun_out/exp_$T.log
done
cp /tmp/libhopf_orig.so paper_1605_01799_b200/libhopf.so
