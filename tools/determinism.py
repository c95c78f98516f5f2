"""Run the same Algorithm 1 / Lloyd passes twice (fresh handles) and report the
first pass whose (energy, changed, accepted) differ. usage: determinism.py CFG PASSES [lloyd|aa] [bounded]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfg, P = sys.argv[1], int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "lloyd"
bounded = len(sys.argv) > 4 and sys.argv[4] == "bounded"
X, C0, c = synthetic.make(cfg)
Xd = torch.from_numpy(X).cuda()
runs = []
for rep in range(2):
    if rep == 1:                                   # hand the next workspace garbage, not the first run's bytes
        junk = torch.randint(-2**31, 2**31 - 1, (int(2.5e9) // 4,), dtype=torch.int32, device="cuda")
        del junk
    kw = dict(m0=0, dynamic_m=False) if mode == "lloyd" else dict(m0=c.m0)
    km = aakm.KMeans(Xd, c.K, aakm.config(bounded=bounded, **kw))
    tr = [km.aa_step(torch.from_numpy(C0).cuda())]
    for _ in range(P):
        r = km.aa_step()
        tr.append(r)
        if r["converged"]:
            break
    km.close()
    runs.append(tr)
a, b = runs
for i, (x, y) in enumerate(zip(a, b)):
    kx = (x["energy"], x["changed"], x["accepted"], x["m"])
    ky = (y["energy"], y["changed"], y["accepted"], y["m"])
    if kx != ky:
        print(f"first difference at pass {i}: {kx} vs {ky}")
        break
else:
    print(f"identical over {min(len(a), len(b))} passes; lengths {len(a)} {len(b)}")
