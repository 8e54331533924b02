#!/bin/bash
TAG=${1:-p}; CFG=${2:-c3}
mkdir -p gpurun_out
bash tools/gpu_ncu_one.sh $TAG $CFG 100000 hopf_diag
ncu -i gpurun_out/prof_${CFG}_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${CFG}_$TAG.csv 2>&1
