mkdir -p gpurun_out
./tools/tcgen05_probe/probe > gpurun_out/probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/probe.log
for C in c3 c2 c5; do timeout 300 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_r01g.log 2>&1; done
