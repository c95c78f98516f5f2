"""Tiny end-to-end runs of every engine for compute-sanitizer:
c1 (SIMT), c2 (SIMT, atomic update), a c3-shaped 3xTF32 shard, a c5-shaped
2xFP16 shard (dense and bounded, label-sorted update with gather4), K-Means++
and the API calls.  usage: python tools/sanitize_run.py [which ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1805_10638_b200 import aakm, synthetic

which = sys.argv[1:] or ["c1", "c2", "tc", "tc16", "bounded", "seed"]
for w in which:
    if w in ("c1", "c2"):
        X, C0, c = synthetic.make(w, N=4000 if w == "c2" else None)
        km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(m0=5, max_iters=30))
    elif w == "tc":
        X, C0, c = synthetic.make("c3", N=70_000, K=64)
        km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(m0=5, max_iters=6, assign_path="tc"))
    elif w in ("tc16", "bounded"):
        X, C0, c = synthetic.make("c5", N=70_000, K=256)
        km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K,
                         aakm.config(m0=5, max_iters=6, assign_path="tc16", bounded=(w == "bounded")))
    elif w == "seed":
        X, C0, c = synthetic.make("c4", N=20_000, K=32)
        km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config())
        Cs, idx = km.seed_pp(synthetic.seed_uniforms("c4", c.K))
        km.close()
        print(w, "seed ok", idx[:4])
        continue
    C, lab, rep = km.run(torch.from_numpy(C0).cuda())
    lab2, E, ch = km.assign(C, labels_prev=lab)
    G, cnt = km.update(lab2, C)
    km.aa_step(torch.from_numpy(C0).cuda())
    for _ in range(3):
        km.aa_step()
    torch.cuda.synchronize()
    print(w, km.path, "iters", rep["iters"], "E", rep["energy"], "changed", ch)
    km.close()
