# A/B of two builds (abtmp/libaakm_{A,B}.so) on the SIMT assignment (c1, c2 full size)
cp paper_1805_10638_b200/libaakm.so abtmp/libaakm_cur.so
for r in 1 2; do for v in A B; do
  cp abtmp/libaakm_$v.so paper_1805_10638_b200/libaakm.so
  echo -n "$v: "; python tools/probe_tc.py simt 100000 c2 | tail -1
  echo -n "$v: "; python tools/probe_tc.py simt 10000 c1 | tail -1
done; done
cp abtmp/libaakm_cur.so paper_1805_10638_b200/libaakm.so
