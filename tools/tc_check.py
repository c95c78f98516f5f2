"""Quick check of the tensor-core assignment engine vs the oracle and the SIMT engine."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import oracle
from paper_1805_10638_b200 import aakm, synthetic
for cfg, N in [("c3", 30011), ("c4", 8003), ("c5", 8009), ("c5", 200000)]:
    X, C0, c = synthetic.make(cfg, N=N)
    Xd = torch.from_numpy(X).cuda()
    out = {}
    for path in (("tc", "tc16", "simt") if c.d in (64, 128) else ("tc", "simt")):
        km = aakm.KMeans(Xd, c.K, aakm.config(assign_path=path))
        lab, E, _ = km.assign(torch.from_numpy(C0).cuda())
        torch.cuda.synchronize()
        t0 = time.time()
        for _ in range(3):
            lab, E, _ = km.assign(torch.from_numpy(C0).cuda())
        torch.cuda.synchronize()
        dt = (time.time() - t0) / 3
        out[path] = (lab.cpu().numpy(), E, km.last_flagged(), dt, km.path)
        km.close()
    n_check = min(N, 8009)
    ref = oracle.assign(X[:n_check], C0.astype(np.float64))
    for path, (lab, E, fl, dt, p) in out.items():
        mism = int((lab[:n_check] != ref).sum())
        print(f"{cfg} N={N} {p}: mismatches={mism}/{n_check} flagged={fl} ({fl/N:.2e}) E={E:.6e} t={dt*1e3:.2f} ms")
