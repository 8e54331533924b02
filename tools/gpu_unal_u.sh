#!/bin/bash
# K4g on unaligned rows vs the register union kernel (C5 law at n = 63 / 64 / 65)
for n in 63 64 65; do
  for E in "X=1" "HOPF_UNION_TMG=0"; do
    env $E python bench.py --config c5 --n $n --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 n=$n $E', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['roofline'].get('kernel'))"
  done
done
