#!/bin/bash
# A/B the assignment launch of two builds (abtmp/libaakm_A.so, abtmp/libaakm_B.so), alternating
cp paper_1805_10638_b200/libaakm.so abtmp/libaakm_cur.so
for r in 1 2; do
  for v in A B; do
    cp abtmp/libaakm_$v.so paper_1805_10638_b200/libaakm.so
    echo -n "$v: "; python tools/probe_tc.py auto 4000000 ${1:-c5} | tail -1
  done
done
cp abtmp/libaakm_cur.so paper_1805_10638_b200/libaakm.so
