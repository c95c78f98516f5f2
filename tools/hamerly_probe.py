"""How many rows would a Hamerly-bounded assignment skip?  Runs Algorithm 1 (or Lloyd)
on a c5/c4 variant through the GPU path, exports each assigned centroid set, and tracks
per-row Hamerly bounds (ub += shift of own centroid, lb -= max shift) in torch fp64,
printing the fraction of rows proven unchanged per pass."""
import sys, torch
sys.path.insert(0, '.')
from paper_1805_10638_b200 import aakm, synthetic
cfg = sys.argv[1]; N = int(sys.argv[2]); m0 = int(sys.argv[3]); passes = int(sys.argv[4])
X, C0, c = synthetic.make(cfg, N=N)
Xd = torch.from_numpy(X).cuda()
km = aakm.KMeans(Xd, c.K, aakm.config(m0=m0, dynamic_m=m0 > 0))
km.aa_step(torch.from_numpy(C0).cuda(), info=False)
X64 = Xd.double(); xn = (X64 * X64).sum(1)
def top2(C):
    C64 = torch.as_tensor(C).cuda().double()
    D = (xn[:, None] - 2 * X64 @ C64.T + (C64 * C64).sum(1)[None, :]).clamp_min(0).sqrt()
    v, i = torch.topk(D, 2, dim=1, largest=False)
    return v[:, 0], v[:, 1], i[:, 0], C64
ub = lb = lab = Cref = None
for p in range(passes):
    s = km.state_export(); C = s["C"]          # the iterate the next pass assigns first
    d1, d2, a, C64 = top2(C)
    if ub is not None:
        sh = (C64 - Cref).norm(dim=1); D = sh.max()
        ub2 = ub + sh[lab]; lb2 = lb - D
        safe = ub2 < lb2
        ok = (a[safe] == lab[safe]).all().item()
        print(f"pass {p}: max shift {D.item():.3e}  safe {safe.float().mean().item():.3f}  changed {(a != lab).float().mean().item():.4f}  bound-consistent {ok}")
        ub = torch.where(safe, ub2, d1); lb = torch.where(safe, lb2, d2)
    else:
        ub, lb = d1, d2
    lab, Cref = a, C64
    info = km.aa_step()
    if info["converged"]:
        print("converged at", p); break
