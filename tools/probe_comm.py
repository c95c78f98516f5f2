"""Per-pass time of Algorithm 1 on one GPU with no communicator, with a 1-rank
communicator (ncclAllReduce of the packed vector), and with the f4 fused
combine (symmetric window + device barriers); prints the fused transport mode.
usage: probe_comm.py [cfg] [passes]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 20
X, C0, c = synthetic.make(cfg, seed=0)
Xd, C0d = torch.from_numpy(X).cuda(), torch.from_numpy(C0).cuda()
for name, kw in [("none", {}), ("nccl_allreduce", dict(comm_always=True)),
                 ("fused", dict(comm_always=True, fused_comm=True))]:
    km = aakm.KMeans(Xd, c.K, aakm.config(m0=5, **kw))
    km.aa_step(C0d, info=False)
    for _ in range(3):
        km.aa_step(info=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(km.stream)
    for _ in range(P):
        km.aa_step(info=False)
    e1.record(km.stream)
    torch.cuda.synchronize()
    print(json.dumps({"config": cfg, "variant": name, "comm_info": km.comm_info(), "ms_per_pass": e0.elapsed_time(e1) / P}))
    km.close()
