#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py, one tool x engine per process (logs in gpurun_out/sanitize/)
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck initcheck; do
  for w in c1 c2 tc tc16 bounded seed; do
    timeout 400 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 python tools/sanitize_run.py $w \
      > gpurun_out/sanitize/${tool}_${w}.log 2>&1
    echo "$tool $w rc=$?" >> gpurun_out/sanitize/summary.txt
  done
done
