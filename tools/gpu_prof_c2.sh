#!/bin/bash
TAG=${1:-p}
mkdir -p gpurun_out
bash tools/gpu_ncu_one.sh $TAG c2 1000000 hopf_diag
ncu -i gpurun_out/prof_c2_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_c2_$TAG.csv 2>&1
