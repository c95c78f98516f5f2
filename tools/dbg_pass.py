import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1805_10638_b200 import aakm, synthetic
X, C0, c = synthetic.make(sys.argv[1] if len(sys.argv) > 1 else "c1")
km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(m0=5))
print(km.aa_step(torch.from_numpy(C0).cuda()))
for i in range(3):
    print(km.aa_step())
