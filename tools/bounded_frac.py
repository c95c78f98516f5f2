"""Rows scored by the bounded engine per window of passes (late-run behaviour).
usage: bounded_frac.py CFG WINDOW NWIN"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfg, W, NW = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
X, C0, c = synthetic.make(cfg)
km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(m0=c.m0, bounded=True))
km.aa_step(torch.from_numpy(C0).cuda(), info=False)
prev = km.bounded_stats()
for w in range(NW):
    rej = 0
    for _ in range(W):
        r = km.aa_step()
        rej += r["rejected"]
        if r["converged"]:
            break
    cur = km.bounded_stats()
    print(f"passes {w * W}-{(w + 1) * W}: scored {(cur[0] - prev[0]) / max(cur[1] - prev[1], 1):.3f}, "
          f"rejected {rej}, flagged(last) {km.last_flagged()}, m {r['m']}, changed {r['changed']}", flush=True)
    prev = cur
    if r["converged"]:
        break
km.close()
