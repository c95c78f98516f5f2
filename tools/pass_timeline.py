"""CUPTI kernel timeline (torch.profiler) of Algorithm 1 passes: per-kernel
durations and the gaps between them, eager (kmeans_aa_step) and graph-replayed
(kmeans_run).  usage: pass_timeline.py cfg [passes]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import collections, torch
from torch.profiler import profile, ProfilerActivity
from paper_1805_10638_b200 import aakm, synthetic

cfg = sys.argv[1]; P = int(sys.argv[2]) if len(sys.argv) > 2 else 5
bounded = len(sys.argv) > 3 and sys.argv[3] == "bounded"
WARM = int(sys.argv[4]) if len(sys.argv) > 4 else 3
X, C0, c = synthetic.make(cfg, seed=0)
Xd, C0d = torch.from_numpy(X).cuda(), torch.from_numpy(C0).cuda()
km = aakm.KMeans(Xd, c.K, aakm.config(m0=5, bounded=bounded))
km.aa_step(C0d, info=False)
for _ in range(WARM):
    km.aa_step(info=False)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(P):
        km.aa_step(info=False)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
span = (evs[-1].time_range.end - evs[0].time_range.start) / P
busy = sum(e.time_range.elapsed_us() for e in evs) / P
agg = collections.defaultdict(lambda: [0.0, 0])
for e in evs:
    k = e.name.split("(")[0].replace("void ", "").replace("aakm::", "")[:34]
    agg[k][0] += e.time_range.elapsed_us() / P; agg[k][1] += 1
print(f"{cfg} eager: {len(evs) / P:.1f} kernels/pass, span {span:.1f} us/pass, busy {busy:.1f} us/pass")
for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:34s} {t:8.2f} us/pass  x{n / P:.1f}")
print("last pass, in order (kernel, duration, gap before it):")
per = len(evs) // P
last = None
for e in evs[-per:]:
    gap = e.time_range.start - last if last is not None else 0.0
    print(f"  {e.name.split('(')[0].replace('void ', '').replace('aakm::', '')[:34]:34s} {e.time_range.elapsed_us():9.2f} {gap:7.2f}")
    last = e.time_range.end
km.close()
