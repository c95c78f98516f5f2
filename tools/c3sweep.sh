# c3 assignment probes (AAKM_TC_DBG bits, see probe_tc.py / assign_tc.cu)
for dbg in 0 256 2 258; do AAKM_TC_DBG=$dbg python tools/probe_tc.py auto 4000000 c3; done
