"""Update-step probe: the label-sorted update of one G-evaluation
(k_hist, k_scan_a/b, k_scatter, k_segsum_bulk) timed in-stream through
kmeans_update_partials on a full-size config, with a CUPTI kernel timeline
(torch.profiler) to show per-kernel durations and the gaps between them.
usage: probe_update.py [cfg] [reps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1805_10638_b200 import aakm, synthetic

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
X, C0, c = synthetic.make(cfg, seed=0)
Xd = torch.from_numpy(X).cuda()
km = aakm.KMeans(Xd, c.K, aakm.config(m0=5))
C = torch.from_numpy(C0.astype(np.float64)).cuda()
lab, _, _ = km.assign(C)
C1 = C + 0.01
prev = lab.clone()
lab2, _, _ = km.assign(C1)
if os.environ.get("PROBE_SEQ"):              # labels in contiguous row blocks: the gathers become sequential
    lab2 = (torch.arange(c.N, device="cuda", dtype=torch.int64) * c.K // c.N).to(torch.int32)
for _ in range(3):
    km.update_partials(lab2, C1, labels_prev=prev)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(km.stream)
for _ in range(reps):
    km.update_partials(lab2, C1, labels_prev=prev)
e1.record(km.stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
gb = (c.N * c.d * 4 + c.N * 4) / 1e9
print(json.dumps({"config": cfg, "update_partials_ms": ms, "algorithmic_GB": gb, "GBps": gb / (ms / 1e3)}))
try:
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            km.update_partials(lab2, C1, labels_prev=prev)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    last = None
    for e in evs[-12:]:
        gap = (e.time_range.start - last) if last is not None else 0
        print(f"  {e.name[:40]:40s} dur {e.time_range.elapsed_us():8.1f} us  gap {gap:6.1f} us")
        last = e.time_range.end
except Exception as ex:
    print("profiler unavailable:", ex)
km.close()
