"""Summarise an AAKM_TC_TRACE stamp file (tc_stamp events of CTAs 0/1 of the
tensor-core assignment; build with AAKM_NVCC_EXTRA=-DAAKM_TC_TRACE_BUILD).
Events: 0 split done, 1 MMA sees operands, 2 MMA sees accumulator free,
3 MMA commit issued, 4 epilogue sees accumulator, 5 epilogue done,
6 splitter X landed, 7 splitter operand buffer free.  usage: trace_tc.py FILE"""
import sys
import numpy as np

rows = np.loadtxt(sys.argv[1], dtype=np.float64)
for b in (0, 1):
    r = rows[rows[:, 0] == b]
    ev = r[:, 2:]
    live = ev[:, 5] > 0
    ev = ev[live]
    n = len(ev)
    if n < 4:
        continue
    t0 = ev[:, [0, 4, 5, 6, 7] + ([1, 2, 3] if b == 0 else [])].min()
    e = (ev - t0) / 1e3
    def med(x):
        return float(np.median(x[1:-1])) if len(x) > 2 else float('nan')
    out = {
        "tiles": n,
        "period": med(np.diff(e[:, 5])),
        "first_epi_done": float(e[0, 5]),
        "split": med(e[:, 0] - np.maximum(e[:, 6], e[:, 7])),
        "split_wait_opbuf": med(e[:, 7] - e[:, 6]),
        "epi_busy": med(e[:, 5] - e[:, 4]),
        "epi_wait_acc": med(e[1:, 4] - e[:-1, 5]),
    }
    if b == 0:
        out.update({
            "mma_wait_ops": med(e[:, 1] - np.concatenate([[0], e[:-1, 3]])),
            "mma_issue": med(e[:, 3] - np.maximum(e[:, 1], e[:, 2])),
            "mma_to_epi": med(e[:, 4] - e[:, 3]),
            "op_ready_to_mma": med(e[:, 1] - e[:, 0]),
            "accfree_after_ops": med(e[:, 2] - e[:, 1]),
        })
    print(b, {k: round(v, 3) if isinstance(v, float) else v for k, v in out.items()})
    if b == 0:
        for i in (0, 1, 2, 3, n // 2, n - 1):
            print("   it", i, " ".join(f"{x:8.2f}" for x in e[i]))
