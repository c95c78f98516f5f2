#!/bin/bash
# usage: tools/launches.sh c4 c3 ...   (ncu launch lists of a short bench run per config)
for c in "$@"; do
  CMD="python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --ttc-config none --seed-config none"
  $CMD > gpurun_out/plain_$c.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv $CMD > gpurun_out/ncu_launch_$c.log 2>&1
done
