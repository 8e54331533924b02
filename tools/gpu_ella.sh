#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ellA" 2>&1 | tail -25 > gpurun_out/ella_tests.log
timeout 300 python bench.py --config t4a --steps 5 --warmup 3 > gpurun_out/ella_bench.json 2> gpurun_out/ella_bench.err
cat gpurun_out/ella_tests.log; cat gpurun_out/ella_bench.json | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l); r = d.get('roofline') or {}
        print(d['config']['workload'], d['value'], d['ms_per_step'], r.get('kernel'), r.get('frac'), r.get('mean_iters'), d.get('cpu_baseline', {}).get('value'), (d.get('e2e') or {}).get('value'))
"
tail -5 gpurun_out/ella_bench.err
