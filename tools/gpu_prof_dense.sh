#!/bin/bash
TAG=${1:-p}
mkdir -p gpurun_out
bash tools/gpu_ncu_one.sh $TAG c4 200000 hopf_dense_tc
ncu -i gpurun_out/prof_c4_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_c4_$TAG.csv 2>&1
ncu -i gpurun_out/prof_c4_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_c4_$TAG.csv 2>&1
