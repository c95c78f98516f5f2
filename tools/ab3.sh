# A/B/C of three builds (abtmp/libaakm_{A,B,C}.so) on one box: probe_tc on the given configs
cp paper_1805_10638_b200/libaakm.so abtmp/libaakm_cur.so
for r in 1 2; do for c in "$@"; do for v in A B C; do
  [ -f abtmp/libaakm_$v.so ] || continue
  cp abtmp/libaakm_$v.so paper_1805_10638_b200/libaakm.so
  echo -n "$v: "; python tools/probe_tc.py auto 4000000 $c 2>&1 | grep -v Warn | tail -1
done; done; done
cp abtmp/libaakm_cur.so paper_1805_10638_b200/libaakm.so
