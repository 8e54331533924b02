#!/bin/bash
# quick A/B: selected GPU tests and bench lines (ms_per_step and roofline fraction)
# usage: tools/gpu_quick.sh "<pytest -k expr>" cfg1 cfg2 ...
K="$1"; shift
if [ -n "$K" ]; then python -m pytest tests -q -m gpu -k "$K" -x 2>&1 | tail -3; fi
for c in "$@"; do
  python bench.py --config $c --steps 30 --warmup 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), d['roofline'].get('kernel'))"
done
