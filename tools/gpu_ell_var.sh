#!/bin/bash
# c2e under each candidate ELL variant
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in "$@"; do
  HOPF_DIAG_VARIANT=$v timeout 300 python bench.py --config c2e --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); r = d['roofline']; print('$v', d['ms_per_step'], r['frac'])"
done
