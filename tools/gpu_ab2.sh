#!/bin/bash
# c2 / c2h with the current build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in c2 c2h c2 c2h; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); r = d['roofline']; print('$c', d['ms_per_step'], r['frac'])"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "wl1 or c2 or maxh" 2>&1 | tail -2
