#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "union or distance or counter or c5" 2>&1 | tail -3
for v in "$@"; do
  for c in c5 c5d; do
  HOPF_DIAG_VARIANT=$v timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$v $c', d['ms_per_step'], d['roofline']['frac'])"
  done
done
