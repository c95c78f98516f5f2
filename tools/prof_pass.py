"""Per-kernel breakdown of Algorithm 1 passes (run with AAKM_PROFILE=1)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1805_10638_b200 import aakm, synthetic
cfg = sys.argv[1]; passes = int(sys.argv[2]) if len(sys.argv) > 2 else 4
path = sys.argv[3] if len(sys.argv) > 3 else "auto"
bounded = len(sys.argv) > 4 and sys.argv[4] == "bounded"
warm = int(sys.argv[5]) if len(sys.argv) > 5 else 0
X, C0, c = synthetic.make(cfg)
km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(m0=5, assign_path=path, bounded=bounded))
km.aa_step(torch.from_numpy(C0).cuda(), info=False)
for _ in range(warm):
    km.aa_step(info=False)
for _ in range(passes):
    info = km.aa_step()
print(cfg, km.path, "flagged(last)", km.last_flagged(), info)
km.close()
