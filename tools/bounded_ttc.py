"""Time to converge (or a fixed pass budget) with and without the Hamerly-bounded
assignment (cfg.bounded), same data and C^0; prints JSON lines."""
import json, sys, torch
sys.path.insert(0, '.')
from paper_1805_10638_b200 import aakm, synthetic
cfg = sys.argv[1]; variant = sys.argv[2]; max_iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
X, C0, c = synthetic.make(cfg)
Xd = torch.from_numpy(X).cuda(); C0d = torch.from_numpy(C0).cuda()
kw = dict(m0=0, dynamic_m=False) if variant == "lloyd" else dict(m0=c.m0)
for bounded in (False, True):
    km = aakm.KMeans(Xd, c.K, aakm.config(max_iters=max_iters, bounded=bounded, **kw))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(km.stream)
    C, lab, rep = km.run(C0d)
    e1.record(km.stream); torch.cuda.synchronize()
    sc, tot = km.bounded_stats()
    print(json.dumps({"config": cfg, "variant": variant, "bounded": bounded, "seconds": e0.elapsed_time(e1) / 1e3,
                      "iters": rep["iters"], "n_assign": rep["n_assign"], "converged": bool(rep["converged"]),
                      "energy": rep["energy"], "rows_scored_frac": sc / max(tot, 1)}), flush=True)
    km.close()
