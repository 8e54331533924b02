#!/bin/bash
# K1g on unaligned rows vs the register kernel (C2 law, n around 100, and C3 law at n = 255 / 257)
for n in 99 100 101; do
  for E in "X=1" "HOPF_DIAG_TMG=0"; do
    env $E python bench.py --config c2 --n $n --steps 20 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 n=$n $E', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['roofline'].get('kernel'))"
  done
done
