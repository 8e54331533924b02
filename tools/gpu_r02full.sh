#!/bin/bash
# round-2 evidence run: tests, smoke, every bench line, launch lists, ncu --set full of the top kernels
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default_$TAG.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_$TAG.log
for C in c2 c5 c4 c1 c5d c2h c2e c2i t5 t4a; do
  timeout 600 python bench.py --config $C --steps 20 --warmup 3 > gpurun_out/bench_${C}_$TAG.log 2>&1
  echo "rc=$?" >> gpurun_out/bench_${C}_$TAG.log
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
for C in c2 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${C}_$TAG.csv python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$TAG.csv python bench.py --config c4 --M 200000 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
bash tools/gpu_ncu_src.sh $TAG c3 100000 hopf_diag_tm
bash tools/gpu_ncu_src.sh $TAG c2 1000000 hopf_diag_tmg
bash tools/gpu_ncu_src.sh $TAG c5 500000 hopf_union_tmg
bash tools/gpu_ncu_src.sh $TAG c4 200000 hopf_dense_tc3
echo done > gpurun_out/done_$TAG
