#!/bin/bash
# round-2 check: GPU test suite, smoke, every config benched once
TAG=${1:-r02a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 900 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
for C in c3 c2 c5 c4 c1 c5d c2h c2e c2i t5 t4a; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${C}_$TAG.log 2>&1
  echo "rc=$?" >> gpurun_out/bench_${C}_$TAG.log
done
echo done > gpurun_out/done_$TAG
