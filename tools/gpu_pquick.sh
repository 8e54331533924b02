#!/bin/bash
# a few paper-protocol lines (A/B loop for the small-n kernels); extra args: env settings
for c in p4_id_l1 p4_diag_l1 p8_diag_l2 p12_diag_l1 p16_id_l2 p16_diag_l1 p16_diag_l2; do
  env "${@:-X=1}" python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['roofline'].get('kernel'))"
done
