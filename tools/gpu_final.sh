#!/bin/bash
# final evidence of a round: tools/gpu_r02full.sh, then a randomised parity sweep of every entry point
TAG=${1:-r02f}
bash tools/gpu_r02full.sh $TAG
timeout 400 python tools/fuzz_gpu.py 300 > gpurun_out/fuzz_all_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/fuzz_all_$TAG.log
timeout 300 python tools/fuzz_gpu.py 200 diag > gpurun_out/fuzz_diag_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/fuzz_diag_$TAG.log
