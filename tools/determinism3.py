"""Sequences of kmeans_run variants on one X in one process (state leaking between handles?).
usage: determinism3.py CFG SEQ   e.g. SEQ = aab,aad,aad  (aa/lloyd x b(ounded)/d(ense))"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfg, seq = sys.argv[1], sys.argv[2].split(",")
X, C0, c = synthetic.make(cfg)
Xd = torch.from_numpy(X).cuda()
for v in seq:
    kw = dict(m0=0, dynamic_m=False) if v.startswith("lloyd") else dict(m0=c.m0)
    km = aakm.KMeans(Xd, c.K, aakm.config(bounded=v.endswith("b"), max_iters=20000, **kw))
    _, _, r = km.run(torch.from_numpy(C0).cuda())
    sc, tot = km.bounded_stats()
    km.close()
    print(v, r["iters"], r["energy"], sc / max(tot, 1), flush=True)
print("X unchanged:", bool(torch.equal(Xd.cpu(), torch.from_numpy(X))))
