for dbg in 0 2 4 128 130 6 134 32; do AAKM_TC_DBG=$dbg python tools/probe_tc.py auto 4000000 c3; done
