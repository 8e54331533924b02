#!/bin/bash
# usage: tools/gpu_ncu_src.sh <tag> <config> <M> <kernel-regex> [ENV=VAL]: one ncu --set full capture
TAG=$1; CFG=$2; M=$3; K=$4; ENVV=${5:-X=1}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --M $M --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 env $ENVV $CMD > gpurun_out/plain_${CFG}_$TAG.log 2>&1 && \
timeout 900 env $ENVV ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_${CFG}_$TAG $CMD > gpurun_out/ncu_full_${CFG}_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full_${CFG}_$TAG.log
