#!/bin/bash
# ncu --set full of the dense tc2 kernel (C4, reduced M) and the C3 diag kernel; source pages as csv
TAG=${1:-r01c}
mkdir -p gpurun_out
bash tools/gpu_ncu_one.sh $TAG c4 200000 hopf_dense_tc2
bash tools/gpu_ncu_one.sh $TAG c3 100000 hopf_diag
for C in c4 c3; do
  if [ -f gpurun_out/prof_${C}_$TAG.ncu-rep ]; then
    ncu -i gpurun_out/prof_${C}_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${C}_$TAG.csv 2>&1
    ncu -i gpurun_out/prof_${C}_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_${C}_$TAG.csv 2>&1
  fi
done
echo done > gpurun_out/done_$TAG
