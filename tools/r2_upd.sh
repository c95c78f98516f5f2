#!/bin/bash
# update-engine probes: full, data-movement only (dbg 8), sums without energy (dbg 64)
mkdir -p gpurun_out
for cfg in c5 c4 c3; do
  for dbg in 0 8 64; do
    AAKM_TC_DBG=$dbg python tools/probe_update.py $cfg 10 2>&1 | head -1 | sed "s/^/dbg=$dbg /" >> gpurun_out/upd_probe.txt
  done
done
