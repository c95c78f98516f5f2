cp paper_1805_10638_b200/libaakm.so /tmp/libaakm_cur.so
for w in "" 2 3 15; do
  cp abtmp/libaakm_trace$w.so paper_1805_10638_b200/libaakm.so
  echo "== epilogue warp ${w:-0}"
  AAKM_TC_TRACE=gpurun_out/trace_c3_w$w.txt python tools/probe_tc.py auto 4000000 c3
  python tools/trace_tc.py gpurun_out/trace_c3_w$w.txt
done
cp /tmp/libaakm_cur.so paper_1805_10638_b200/libaakm.so
