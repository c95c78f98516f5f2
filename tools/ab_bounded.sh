#!/bin/bash
# A/B of two builds (abtmp/libaakm_{A,B}.so) on the bounded engine late in a c4 run
cp paper_1805_10638_b200/libaakm.so abtmp/libaakm_cur.so
for r in 1 2; do
  for v in A B; do
    cp abtmp/libaakm_$v.so paper_1805_10638_b200/libaakm.so
    echo -n "$v: "; python tools/bounded_assign_probe.py ${1:-c4} ${2:-1200} ${3:-40} | tail -1
  done
done
cp abtmp/libaakm_cur.so paper_1805_10638_b200/libaakm.so
