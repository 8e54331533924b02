#!/bin/bash
# grouped TMEM kernel vs register kernel over n (A/B by HOPF_DIAG_TMG=0), C2 law (wl1) and C3 law (l2)
TAG=$1; shift
mkdir -p gpurun_out
: > gpurun_out/nsweep_$TAG.txt
for CFG in c2 c3; do for N in "$@"; do
  M=$(( 100000000 / N ))
  for V in "X=1" "HOPF_DIAG_TMG=0"; do
    timeout 300 env $V python bench.py --config $CFG --n $N --M $M --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ns_$TAG.log 2>&1
    echo "$CFG n=$N M=$M $V $(grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/ns_$TAG.log) $(grep -h -o '"kernel": "[^"]*"' gpurun_out/ns_$TAG.log) $(grep -h -o '"frac": [0-9.]*' gpurun_out/ns_$TAG.log | head -1)" >> gpurun_out/nsweep_$TAG.txt
  done
done; done
