#!/bin/bash
# usage: tools/gpu_libab.sh <config> <lib1> [lib2 ...]: bench one config with each library build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
CFG=$1; shift
cp paper_1605_01799_b200/libhopf.so /tmp/libhopf_default.so
for L in default "$@"; do
  if [ "$L" = default ]; then cp /tmp/libhopf_default.so paper_1605_01799_b200/libhopf.so; else cp "$L" paper_1605_01799_b200/libhopf.so; fi
  touch paper_1605_01799_b200/libhopf.so
  timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$L', d['ms_per_step'], d['roofline']['frac'])"
done
cp /tmp/libhopf_default.so paper_1605_01799_b200/libhopf.so
