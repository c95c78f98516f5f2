"""Time to converge with and without the incremental update (AAKM_DELTA_DIV,
read at create): Algorithm 1 (m0 = 5, dynamic) and Lloyd on a full-size config,
CUDA events; prints seconds, iterations and kmeans_update_stats.
usage: ttc_delta.py cfg div[,div...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
divs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "64"]
X, C0, c = synthetic.make(cfg)
Xd, C0d = torch.from_numpy(X).cuda(), torch.from_numpy(C0).cuda()
for div in divs:
    os.environ["AAKM_DELTA_DIV"] = div
    for name, kw in (("aa", dict(m0=c.m0, dynamic_m=True)), ("lloyd", dict(m0=0, dynamic_m=False))):
        km = aakm.KMeans(Xd, c.K, aakm.config(max_iters=10000, bounded=c.d in (64, 128), **kw))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        C, lab, rep = km.run(C0d)
        e1.record()
        torch.cuda.synchronize()
        ne, ni, moved = km.update_stats()
        print(json.dumps({"config": cfg, "variant": name, "delta_div": int(div), "seconds": e0.elapsed_time(e1) / 1e3,
                          "iters": rep["iters"], "n_assign": rep["n_assign"], "energy": rep["energy"],
                          "evals": ne, "incremental": ni, "rows_moved": moved}), flush=True)
        km.close()
