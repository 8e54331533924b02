#!/bin/bash
# compute-sanitizer over every kernel family (small inputs); logs to gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for T in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$T.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$T.log
done
