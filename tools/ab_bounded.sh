# A/B of two builds (abtmp/libaakm_{A,B}.so) on bounded kmeans_run timelines (c4)
cp paper_1805_10638_b200/libaakm.so abtmp/libaakm_cur.so
for r in 1 2; do for v in A B; do
  cp abtmp/libaakm_$v.so paper_1805_10638_b200/libaakm.so
  echo "$v:"; python tools/run_timeline.py ${1:-c4} bounded 2>&1 | grep -E " run: |k_bounds|k_bnd_save|k_shift"
done; done
cp abtmp/libaakm_cur.so paper_1805_10638_b200/libaakm.so
