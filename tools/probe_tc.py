"""Time the assignment kernel alone on c5-shaped data (perf probes via AAKM_TC_DBG)."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_1805_10638_b200 import aakm, synthetic
path = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 2_000_000
X, C0, c = synthetic.make("c5", N=N)
km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(assign_path=path, timing=True))
km.aa_step(torch.from_numpy(C0).cuda(), info=False)
km.assign_timing()
for _ in range(5):
    km.aa_step(None, info=False)
ms, n = km.assign_timing()
print(f"{path} dbg={__import__('os').environ.get('AAKM_TC_DBG','0')} N={N} assign avg {ms/n:.3f} ms -> {2*N*c.K*c.d/(ms/n*1e-3)/1e12:.1f} TF/s")
