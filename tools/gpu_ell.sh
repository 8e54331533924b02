#!/bin/bash
# NEXT-2 ellipsoidal H: parity tests and a c2e bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ell or linf" 2>&1 | tail -15 > gpurun_out/ell_tests.log
timeout 300 python bench.py --config c2e --steps 5 --warmup 3 > gpurun_out/ell_bench.json 2> gpurun_out/ell_bench.err
timeout 300 python bench.py --config c2i --steps 5 --warmup 3 >> gpurun_out/ell_bench.json 2>> gpurun_out/ell_bench.err
timeout 300 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/c2_bench.json 2>> gpurun_out/ell_bench.err
cat gpurun_out/ell_tests.log; cat gpurun_out/ell_bench.json gpurun_out/c2_bench.json | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l); r = d.get('roofline') or {}
        print(d['config']['workload'], d['value'], d['ms_per_step'], r.get('kernel'), r.get('frac'), r.get('mean_iters'))
"
tail -5 gpurun_out/ell_bench.err
