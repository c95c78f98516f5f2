# A/B of two builds (abtmp/libaakm_{A,B}.so) on one box: whole kmeans_run timelines per config
cp paper_1805_10638_b200/libaakm.so abtmp/libaakm_cur.so
for r in 1 2; do for c in "$@"; do for v in A B; do
  cp abtmp/libaakm_$v.so paper_1805_10638_b200/libaakm.so
  echo -n "$v: "; python tools/run_timeline.py $c 2>&1 | grep " run: "
done; done; done
cp abtmp/libaakm_cur.so paper_1805_10638_b200/libaakm.so
