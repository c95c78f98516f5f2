"""CUPTI kernel timeline of a whole graph-replayed kmeans_run (Algorithm 1 to
convergence): kernels per pass, device busy vs span, per-kernel totals.
usage: run_timeline.py cfg [bounded]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import collections, torch
from torch.profiler import profile, ProfilerActivity
from paper_1805_10638_b200 import aakm, synthetic

cfg = sys.argv[1]
bounded = len(sys.argv) > 2 and sys.argv[2] == "bounded"
X, C0, c = synthetic.make(cfg, seed=0)
Xd, C0d = torch.from_numpy(X).cuda(), torch.from_numpy(C0).cuda()
km = aakm.KMeans(Xd, c.K, aakm.config(m0=5, bounded=bounded))
km.run(C0d)                                        # warm (graph capture)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); _, _, rep = km.run(C0d); e1.record(); torch.cuda.synchronize()
wall = e0.elapsed_time(e1)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    _, _, rep = km.run(C0d)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
P = rep["iters"]
span = (evs[-1].time_range.end - evs[0].time_range.start)
busy = sum(e.time_range.elapsed_us() for e in evs)
print(f"{cfg} run: iters {P} n_assign {rep['n_assign']} time {wall:.3f} ms ({wall / P * 1e3:.1f} us/pass); "
      f"profiled span {span / P:.1f} us/pass, busy {busy / P:.1f} us/pass, {len(evs) / P:.1f} kernels/pass")
agg = collections.defaultdict(lambda: [0.0, 0])
for e in evs:
    k = e.name.split("(")[0].replace("void ", "").replace("aakm::", "")[:40]
    agg[k][0] += e.time_range.elapsed_us() / P; agg[k][1] += 1
for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:40s} {t:8.2f} us/pass  x{n / P:.2f}")
gaps = [evs[i + 1].time_range.start - evs[i].time_range.end for i in range(len(evs) - 1)]
gaps.sort()
print(f"  gaps: median {gaps[len(gaps) // 2]:.2f} us, p90 {gaps[int(len(gaps) * .9)]:.2f} us, total {sum(gaps) / P:.1f} us/pass")
km.close()
