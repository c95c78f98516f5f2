"""How many centroids sit inside the near-tie window of each flagged row (c4-type
data): exact fp64 distances on the GPU (torch, chunked) at the centroids of pass P.
usage: tie_stats.py CFG PASSES"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfg, P = sys.argv[1], int(sys.argv[2])
X, C0, c = synthetic.make(cfg)
Xd = torch.from_numpy(X).cuda()
km = aakm.KMeans(Xd, c.K, aakm.config(m0=c.m0))
km.aa_step(torch.from_numpy(C0).cuda(), info=False)
for _ in range(P):
    km.aa_step(info=False)
flag = km.last_flagged()
C = torch.from_numpy(km.state_export()["C"]).cuda().double()
km.close()
cn = (C * C).sum(1)
cmax2 = float(cn.max())
d = c.d
gam = 4 * (3 + 3 * d / 16 + 16) * 2.0 ** -22            # the 2xFP16 window-key bound (DESIGN 5.3), distance units
hist = np.zeros(6, np.int64)
n_flag = 0
for r0 in range(0, c.N, 1 << 17):
    x = Xd[r0:r0 + (1 << 17)].double()
    xn = (x * x).sum(1, keepdim=True)
    D = (xn - 2 * x @ C.T + cn[None]).clamp_min(0)       # fp64, fine for counting
    b = D.min(1, keepdim=True).values
    tau = gam * (xn + cmax2) * 2
    inwin = (D <= b + tau).sum(1)
    f = inwin >= 2
    n_flag += int(f.sum())
    cnt = inwin[f].clamp(max=5).cpu().numpy()
    hist += np.bincount(cnt, minlength=6)
print(f"{cfg} pass {P}: engine flagged {flag}, estimated {n_flag}; rows by #centroids in window:",
      {k: int(v) for k, v in enumerate(hist) if v})
