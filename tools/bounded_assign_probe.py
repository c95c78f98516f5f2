"""Bounded-engine assignment time late in an Algorithm 1 run (bounds prep + MODE 2,
CUDA events via cfg.timing): W passes to warm up, then P timed passes.
usage: bounded_assign_probe.py CFG W P"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfg, W, P = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
X, C0, c = synthetic.make(cfg)
km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(m0=c.m0, bounded=True, timing=True))
km.aa_step(torch.from_numpy(C0).cuda(), info=False)
for _ in range(W):
    km.aa_step(info=False)
km.assign_timing()
s0 = km.bounded_stats()
for _ in range(P):
    km.aa_step(info=False)
ms, n = km.assign_timing()
s1 = km.bounded_stats()
km.close()
print(f"{cfg} bounded assign (branch A) avg {ms / max(n, 1):.3f} ms over {n}; scored {(s1[0] - s0[0]) / max(s1[1] - s0[1], 1):.3f}")
