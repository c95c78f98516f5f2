"""Dump per-pass (energy, changed, accepted, m) of eager passes to a .npy (cross-process determinism).
usage: trace_dump.py CFG PASSES lloyd|aa OUT"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfg, P, mode, out = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
X, C0, c = synthetic.make(cfg)
kw = dict(m0=0, dynamic_m=False) if mode == "lloyd" else dict(m0=c.m0)
km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(**kw))
rows = []
r = km.aa_step(torch.from_numpy(C0).cuda())
rows.append((r["energy"], r["changed"], r["accepted"], r["m"]))
for _ in range(P):
    r = km.aa_step()
    rows.append((r["energy"], r["changed"], r["accepted"], r["m"]))
    if r["converged"]:
        break
np.save(out, np.array(rows, dtype=np.float64))
print(out, len(rows))
