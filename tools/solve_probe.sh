cp paper_1805_10638_b200/libaakm.so /tmp/cur.so; cp abtmp/libaakm_solve.so paper_1805_10638_b200/libaakm.so
for a in "c3 50" "c3 300" "c3 800" "c2 40" "c5 30"; do AAKM_TC_TRACE=/tmp/x AAKM_SOLVE_TRACE=/tmp/sv python tools/solve_probe.py $a; done
cp /tmp/cur.so paper_1805_10638_b200/libaakm.so
