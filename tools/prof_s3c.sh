for dbg in 0 256 4 260 0; do AAKM_TC_DBG=$dbg python tools/probe_tc.py auto 4000000 c4 2>&1 | grep -v Warn; done
for dbg in 0 256; do AAKM_TC_DBG=$dbg python tools/probe_tc.py auto 4000000 c5 2>&1 | grep -v Warn; done
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_assign_tc<.int.1, .int.0,' -s 2 -c 1 -o gpurun_out/s3_c3_assign python tools/probe_tc.py auto 1000000 c3 > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_assign_tc<.int.4, .int.0,' -s 2 -c 1 -o gpurun_out/s3_c4_assign python tools/probe_tc.py auto 4000000 c4 > gpurun_out/ncu_c4.log 2>&1
