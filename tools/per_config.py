"""SURVEY 8(d.4) per-config metrics on one GPU: for c1..c5 (full sizes), W warm-up
passes then P timed Algorithm 1 passes (eager, CUDA events around the loop);
assignment launch time from kmeans_assign_timing; dist-evals/s of the
assignment and of the whole pass; % of the engine's roofline.
usage: per_config.py [cfgs] [P] [W]   -> one JSON line per config"""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_10638_b200 import aakm, synthetic

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "c3", "c4", "c5"]
P = int(sys.argv[2]) if len(sys.argv) > 2 else 20
W = int(sys.argv[3]) if len(sys.argv) > 3 else 3
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
bf16 = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
bf16_burst = peaks["bf16_tflops"]
for cfg in cfgs:
    X, C0, c = synthetic.make(cfg)
    km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(m0=c.m0, timing=True))
    km.aa_step(torch.from_numpy(C0).cuda(), info=False)
    for _ in range(W):
        km.aa_step(info=False)
    st0 = km.state_export()["n_assign"]
    km.assign_timing()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(km.stream)
    for _ in range(P):
        km.aa_step(info=False)
    e1.record(km.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    na = km.state_export()["n_assign"] - st0
    a_ms, a_n = km.assign_timing()
    path = km.path
    km.close()
    t_a = a_ms / max(a_n, 1)
    flops = 2.0 * c.N * c.K * c.d / (t_a / 1e3) / 1e12
    peak = {"tc16": bf16 / 3.0, "tc": bf16 * (1.1 / 2.25) / 3.0}.get(path, 148 * 128 * 2 * 1965e6 / 1e12)
    peak_b = {"tc16": bf16_burst / 3.0, "tc": bf16_burst * (1.1 / 2.25) / 3.0}.get(path, peak)
    print(json.dumps({"config": cfg, "N": c.N, "d": c.d, "K": c.K, "path": path, "passes": P, "n_assign": na,
                      "ms_per_pass": ms / P, "assign_ms": t_a, "assign_dist_evals_per_s": c.N * c.K / (t_a / 1e3),
                      "pass_dist_evals_per_s": c.N * c.K * na / (ms / 1e3),
                      "assign_tflops_fp32eq": flops, "peak_tflops": peak, "roofline_frac": flops / peak,
                      "peak_tflops_burst": peak_b, "roofline_frac_burst": flops / peak_b}), flush=True)
