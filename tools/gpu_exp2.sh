#!/bin/bash
# C4 bench for each alternative build under exp/ (the in-tree library is restored afterwards)
mkdir -p gpurun_out
cp paper_1605_01799_b200/libhopf.so /tmp/libhopf_orig.so
for L in exp/libhopf_*.so; do
  T=$(basename $L .so)
  cp $L paper_1605_01799_b200/libhopf.so
  timeout 150 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp2_$T.log 2>&1
  echo rc=$? >> gpurun_out/exp2_$T.log
done
cp /tmp/libhopf_orig.so paper_1605_01799_b200/libhopf.so
