"""Per-rank compute of an R-rank run measured on one GPU: rank 0's shard of the
config (N/R rows, n_global = N), Algorithm 1 passes timed with CUDA events
(eager, after warm-up).  Everything but the allreduce of the packed vector is
what each rank runs, so t_1 / (R t_R) bounds the scaling efficiency from above
by the collective's share.  usage: shard_projection.py CFG [R,...] [P]"""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
Rs = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
P = int(sys.argv[3]) if len(sys.argv) > 3 else 20
t1 = None
for R in Rs:
    X, C0, c = synthetic.make_shard(cfg, 0, R, seed=0)
    km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(m0=c.m0), n_global=c.N)
    km.aa_step(torch.from_numpy(C0).cuda(), info=False)
    for _ in range(3):
        km.aa_step(info=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(km.stream)
    for _ in range(P):
        km.aa_step(info=False)
    e1.record(km.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / P
    km.close()
    del X
    torch.cuda.empty_cache()
    if R == 1:
        t1 = ms
    print(json.dumps({"config": cfg, "R": R, "rows_per_rank": c.N // R, "ms_per_pass": ms,
                      "compute_efficiency": (t1 / (R * ms)) if t1 else None}), flush=True)
