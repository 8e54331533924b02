#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for cfg in "3 16" "4 16" "2 32" "3 32" "4 8" "6 8" "3 64"; do
  set -- $cfg
  HOPF_HOST_STREAMS=$1 HOPF_HOST_CHUNK_MB=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$1 $2', d['e2e']['value'], d['ms_per_step'])"
done
