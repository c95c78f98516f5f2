"""kmeans_run twice with FRESH device copies of X (new addresses) and fresh handles:
report iterations/energy of each. usage: determinism2.py CFG [lloyd|aa] [bounded] [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfg = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "lloyd"
bounded = len(sys.argv) > 3 and sys.argv[3] == "bounded"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
X, C0, c = synthetic.make(cfg)
keep = []
for rep in range(reps):
    Xd = torch.from_numpy(X).cuda()
    keep.append(Xd)                                  # distinct addresses every rep
    kw = dict(m0=0, dynamic_m=False) if mode == "lloyd" else dict(m0=c.m0)
    km = aakm.KMeans(Xd, c.K, aakm.config(bounded=bounded, max_iters=20000, **kw))
    _, _, r = km.run(torch.from_numpy(C0).cuda())
    km.close()
    print(rep, r["iters"], r["energy"], flush=True)
