"""f1 cross-check on the CPU oracle: Lloyd vs Algorithm 1 (dynamic m0=5 / m0=2, fixed m=2),
exact fp64 state vs the GPU-mirroring fp32 parity state, on small seeded variants of c2-c5."""
import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import oracle
from paper_1805_10638_b200 import synthetic
for cfg, N, K in [("c2", 100000, 64), ("c3", 30000, 64), ("c5", 20000, 128), ("c4", 20000, 128)]:
    X, C0, c = synthetic.make(cfg, N=N, K=K)
    for name, kw in [("lloyd", dict(m0=0, dynamic_m=False)), ("aa_dyn5", dict(m0=5)), ("aa_dyn2", dict(m0=2)), ("aa_fix2", dict(m0=2, dynamic_m=False))]:
        for parity in (False, True):
            t0 = time.time()
            r = oracle.run(X, C0.astype(np.float64), oracle.OracleConfig(parity=parity, max_iters=3000, **kw))
            print(f"{cfg} N={N} K={K} {name:8s} parity={int(parity)} iters={r['iters']:5d} n_assign={r['n_assign']:5d} rej={r['rejected']:4d} E={r['energy']:.8e} conv={r['converged']} {time.time()-t0:.1f}s", flush=True)
