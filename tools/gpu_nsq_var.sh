#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in "$@"; do
  HOPF_NSQ_VARIANT=$v timeout 300 python bench.py --config t5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); r = d['roofline']; print('$v', d['ms_per_step'], r['frac'], r['mean_iters'])"
done
