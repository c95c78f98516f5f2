"""the CPU oracle timed on this host (OpenMP over all cores):
per config the Assignment-Step on a bounded row sample (dist-evals/s), the
Update and Energy on the same sample, and for c1/c2 Algorithm 1 to convergence
(m0 = 5); c3-c5 full passes are projected from the per-row rates.
One JSON line per config."""
import json
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
from paper_1805_10638_b200 import synthetic

cores = os.cpu_count()
os.environ.setdefault("OMP_NUM_THREADS", str(cores))
for cfg in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "c3", "c4", "c5"]):
    X, C0, c = synthetic.make(cfg)
    C = C0.astype(np.float64)
    rows = int(min(c.N, max(2000, 2.0e9 / (c.K * c.d))))          # ~2e9 sqdist terms
    Xs = np.ascontiguousarray(X[:rows])
    oracle.assign(Xs[:64], C)
    t0 = time.perf_counter(); lab = oracle.assign(Xs, C); ta = time.perf_counter() - t0
    t0 = time.perf_counter(); oracle.update(Xs, lab, C); tu = time.perf_counter() - t0
    t0 = time.perf_counter(); oracle.energy(Xs, C, lab); te = time.perf_counter() - t0
    out = {"config": cfg, "N": c.N, "d": c.d, "K": c.K, "cores": int(os.environ["OMP_NUM_THREADS"]),
           "sample_rows": rows, "assign_s": ta, "assign_dist_evals_per_s": rows * c.K / ta,
           "update_s": tu, "energy_s": te,
           "projected_assign_pass_s": ta * c.N / rows}
    if cfg in ("c1", "c2"):
        t0 = time.perf_counter()
        ref = oracle.run(X, C, oracle.OracleConfig(m0=c.m0))
        out.update({"run_s": time.perf_counter() - t0, "run_iters": ref["iters"], "run_converged": bool(ref["converged"])})
    print(json.dumps(out), flush=True)
