"""Time the assignment kernel alone (forced API assignment, CUDA events around the
launch) on c5-shaped data; perf probes via AAKM_TC_DBG (bit 1: one C tile,
bit 2: no epilogue math, bit 4: no MMAs)."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_1805_10638_b200 import aakm, synthetic
path = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 2_000_000
cfg = sys.argv[3] if len(sys.argv) > 3 else "c5"
X, C0, c = synthetic.make(cfg, N=N)
km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(assign_path=path, timing=True))
Cd = torch.from_numpy(C0).cuda()
km.assign(Cd)
km.assign_timing()
for _ in range(5):
    km.assign(Cd)
ms, n = km.assign_timing()
print(f"{cfg} {km.path} dbg={os.environ.get('AAKM_TC_DBG', '0')} N={N} assign avg {ms / n:.3f} ms -> "
      f"{2 * N * c.K * c.d / (ms / n * 1e-3) / 1e12:.1f} TF/s fp32-equiv, flagged {km.last_flagged()}")
km.close()
