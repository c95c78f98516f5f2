"""f1: Algorithm 1 (dynamic m, m0 = 5 and the paper's default m0 = 2) vs
plain Lloyd (m = 0) vs fixed m = 5 on the BASELINE configs, same seeded data and C^0,
run to convergence (rule R3) on the GPU through kmeans_run (fp64 Anderson state).
The 2xFP16 configs (d in {64, 128}) use the Hamerly-bounded engine (the paper's
pruned Assignment-Step) for every variant, the others the dense one.
Prints one JSON line per run; time = CUDA events around kmeans_run."""
import json, sys, time
sys.path.insert(0, '.')
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "c3", "c4", "c5"]
seeds = [int(s) for s in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
max_iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5000
VARIANTS = {"aa_dynamic_m0_5": dict(m0=5, dynamic_m=True), "aa_dynamic_m0_2": dict(m0=2, dynamic_m=True),
            "lloyd": dict(m0=0, dynamic_m=False), "aa_fixed_m5": dict(m0=5, dynamic_m=False)}
for cfg in cfgs:
    for seed in seeds:
        X, C0, c = synthetic.make(cfg, seed=seed)
        Xd = torch.from_numpy(X).cuda(); C0d = torch.from_numpy(C0).cuda()
        for name, kw in VARIANTS.items():
            bounded = c.d in (64, 128)
            km = aakm.KMeans(Xd, c.K, aakm.config(max_iters=max_iters, bounded=bounded, **kw))
            km.run(C0d) if cfg in ("c1", "c2") else None          # warm (tiny configs: launch/graph setup)
            s = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0.record(s)
            C, lab, rep = km.run(C0d)
            e1.record(s)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            out = {"config": cfg, "seed": seed, "variant": name, "N": c.N, "d": c.d, "K": c.K, "path": km.path + ("+bounded" if bounded else ""),
                   "iters": rep["iters"], "n_assign": rep["n_assign"], "accepted": rep["n_accepted"],
                   "rejected": rep["n_rejected"], "converged": bool(rep["converged"]), "m_final": rep["m_final"],
                   "energy": rep["energy"], "mse": rep["mse"], "seconds_events": e0.elapsed_time(e1) / 1e3,
                   "seconds_wall": wall, "ms_per_assign": 1e3 * e0.elapsed_time(e1) / 1e3 / max(rep["n_assign"], 1)}
            print(json.dumps(out), flush=True)
            km.close()
