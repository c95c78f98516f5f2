"""bench.py -- B200 benchmark of the Anderson-accelerated Lloyd K-Means hot path.

A "step" is one loop pass of Algorithm 1: assignment
(+ near-tie refine), update partials with the fused energy, [NCCL allreduce],
device-side control, fallback G-evaluation when the guard rejects, Gram,
LS solve and mixing -- all rows of SURVEY §8(a) -- on the BASELINE.json
config c5 (N = 16,000,000, d = 64, K = 4096, fp32), sharded over the ranks.

value  = sample-centroid distance evaluations per second of the whole job:
         N * K * (assignment passes performed in the timed steps) / time,
         time = max over ranks of the CUDA-event duration of the K steps.
e2e    = the same metric through the C ABI with HOST inputs: every step copies
         the shard X from pinned host memory to the device, runs the pass and
         reads C^{t+1} and E back.
roofline = the dominant kernel (the assignment engine), algorithmic flops
         2 N K d per launch over its CUDA-event duration inside the timed
         steps, against the tensor (three MMAs per product, fp32-equivalent)
         or FP32 peak.
time_to_converge = Algorithm 1 (bounded and dense assignment) and Lloyd run to
         convergence on --ttc-config (default c4; c5 does not converge within
         5000 passes under Algorithm 1).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5]
       python bench.py --impl reference ...   (the CPU oracle arm)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "assign dist-evals/s (Algorithm 1 passes)"
UNIT = "dist-evals/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


# --------------------------------------------------------------------- clocks
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            try:
                a, b, c = [x.strip() for x in ln.split(",")]
                self.samples.append((float(a), float(b), int(c, 16)))
            except Exception:
                pass

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        load = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        mask = 0
        for s in load:
            mask |= s[2]
        return {"sm_mhz": statistics.median(s[0] for s in load), "sm_max_mhz": max(s[1] for s in load),
                "reasons": [v for k, v in REASONS.items() if mask & k and k != 0x1], "samples": len(load)}


# --------------------------------------------------------------------- multi-rank timing
def max_over_ranks(value, world, device="cuda"):
    """The bench's time of a multi-rank step: the max over ranks of each rank's
    device-timed duration (the contract's "max over ranks"); world == 1: value."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------- oracle arm
def cpu_baseline(X, C0, cfgname, budget_rows=None):
    """The oracle's Assignment-Step (its dominant step) on a bounded row sample."""
    import oracle
    cores = os.cpu_count()
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    K, d = C0.shape
    rows = budget_rows or max(1000, int(4.0e11 / (K * d)))  # ~4e11 fp64 sqdist terms (~10 s on 16 cores)
    rows = min(rows, len(X))
    Xs = np.ascontiguousarray(X[:rows])
    C = C0.astype(np.float64)
    oracle.assign(Xs[:64], C)                                 # warm (build/load)
    t0 = time.perf_counter()
    oracle.assign(Xs, C)
    dt = time.perf_counter() - t0
    return {"value": rows * K / dt, "unit": UNIT, "cores": int(os.environ.get("OMP_NUM_THREADS", cores)),
            "kind": "oracle", "seconds": dt,
            "sample": f"oracle Assignment-Step (fp64 direct differences) of the first {rows} rows of {cfgname} "
                      f"(N={len(X)}, d={d}, K={K}) against C^0"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1805_10638_b200 import synthetic
    X, C0, cfg = synthetic.make(args.config, seed=0)
    K, d = C0.shape
    steps = []
    for _ in range(args.warmup):
        cpu_baseline(X, C0, args.config, budget_rows=2000)
    rows = max(500, int(4.0e9 / (K * d)))                    # ~4e9 fp64 sqdist terms per step (~0.5 s on 16 cores)
    for _ in range(args.steps):
        cb = cpu_baseline(X, C0, args.config, budget_rows=rows)
        steps.append(cb)
    v = statistics.median(s["value"] for s in steps)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(s["seconds"] for s in steps),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: Algorithm 1 passes (m0={cfg.m0}, dynamic m)", "N": cfg.N, "d": cfg.d,
                       "K": cfg.K, "parallelism": "cpu (oracle)",
                       "sample": "each step: the oracle's Assignment-Step (the pass's dominant O(NKd) step) on a row sample"},
            "cpu_baseline": dict(steps[-1], value=v),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------- time to converge
def time_to_converge(cfgname, rank, world, barrier):
    """Algorithm 1 (dynamic m, m0 = 5) with the Hamerly-bounded assignment
    (cfg.bounded, the paper's own pruned Assignment-Step), the same with the
    dense assignment, and plain Lloyd (m = 0, bounded), each run to convergence
    (rule R3) through kmeans_run on the sharded config, C^0 resident; CUDA events
    around the call, max over ranks.  (c5 does not converge within 5000 passes
    under Algorithm 1, see profiles/r01_converge_gpu.jsonl.)"""
    import torch
    import torch.distributed as dist
    from paper_1805_10638_b200 import aakm, synthetic
    X, C0, cfg = synthetic.make_shard(cfgname, rank, world, seed=0)
    Xs = torch.from_numpy(X).cuda()
    C0d = torch.from_numpy(C0).cuda()
    out = {"config": cfgname, "N": cfg.N, "d": cfg.d, "K": cfg.K}
    variants = (("", dict(m0=cfg.m0, bounded=True)), ("dense_", dict(m0=cfg.m0, bounded=False)),
                ("lloyd_", dict(m0=0, dynamic_m=False, bounded=True)))
    for pre, kw in variants:
        km = aakm.KMeans(Xs, cfg.K, aakm.config(max_iters=20000, **kw), n_global=cfg.N, rank=rank, nranks=world)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(km.stream)
        _, _, rep = km.run(C0d)
        e1.record(km.stream)
        barrier()
        sec = max_over_ranks(e0.elapsed_time(e1) / 1e3, world)
        scored, total = km.bounded_stats()
        km.close()
        out.update({pre + "seconds": sec, pre + "iters": rep["iters"], pre + "n_assign": rep["n_assign"],
                    pre + "iterations_per_s": rep["iters"] / max(sec, 1e-9),
                    pre + "converged": bool(rep["converged"]), pre + "energy": rep["energy"],
                    pre + "rows_scored_frac": scored / max(total, 1)})
        if pre == "":
            out.update({"accepted": rep["n_accepted"], "rejected": rep["n_rejected"], "m_final": rep["m_final"],
                        "assign_engine": "bounded 2xFP16" if kw.get("bounded") and cfg.d in (64, 128) else "dense"})
    return out


# --------------------------------------------------------------------- K-Means++ seeding (f3)
E2E_CHUNKS = int(os.environ.get("AAKM_E2E_CHUNKS", "64"))   # 16: 8.60e11, 32: 8.59e11, 64: 8.66e11 (c5)


def seed_pp_bench(cfgname, rank, world, barrier, peaks):
    """kmeans_seed_pp for all K centers of the sharded config (C ABI, X resident),
    CUDA events around the call, max over ranks. Per center one pass over X
    (k_seed_dist: X + D2 read/write) and one over D2 (k_seed_weights): the
    algorithmic bytes are n (4d + 24) per center."""
    import torch
    import torch.distributed as dist
    from paper_1805_10638_b200 import aakm, synthetic
    X, _, cfg = synthetic.make_shard(cfgname, rank, world, seed=0)
    Xs = torch.from_numpy(X).cuda()
    km = aakm.KMeans(Xs, cfg.K, aakm.config(), n_global=cfg.N, rank=rank, nranks=world)
    u = synthetic.seed_uniforms(cfgname, cfg.K)
    barrier()
    L0 = km.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(km.stream)
    _, idx = km.seed_pp(u)
    e1.record(km.stream)
    barrier()
    sec = max_over_ranks(e0.elapsed_time(e1) / 1e3, world)
    launches = km.launch_count() - L0
    km.close()
    n = X.shape[0]
    gbs = cfg.K * n * (4.0 * cfg.d + 24.0) / sec / 1e9
    return {"config": cfgname, "N": cfg.N, "d": cfg.d, "K": cfg.K, "seconds": sec,
            "centers_per_s": cfg.K / sec, "gpu_launches": launches,
            "hbm_gbs_algorithmic": gbs, "hbm_frac": gbs / peaks["hbm_gbs"],
            "first_indices": [int(v) for v in idx[:4]]}


# --------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="auto", choices=["auto", "simt", "tc", "tc16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0, help="e2e timed steps (default: --steps)")
    ap.add_argument("--ttc-config", default="c4", help="config run to convergence for time_to_converge ('none' skips)")
    ap.add_argument("--seed-config", default="c5", help="config seeded by kmeans_seed_pp for seed_pp ('none' skips)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_1805_10638_b200 import aakm, synthetic

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    X, C0, cfg = synthetic.make_shard(args.config, rank, world, seed=0)     # this rank's rows only
    lo, hi = synthetic.shard_bounds(cfg.N, rank, world)
    Xs = torch.from_numpy(X).cuda()
    X_host = torch.from_numpy(X).pin_memory()
    C0d = torch.from_numpy(C0).cuda()
    km = aakm.KMeans(Xs, cfg.K, aakm.config(m0=cfg.m0, assign_path=args.path, timing=True, x_refresh=True),
                     n_global=cfg.N, rank=rank, nranks=world)
    stream = km.stream

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # Algorithm 1 line 1, then warm-up passes (untimed)
    km.aa_step(C0d, info=False)
    for _ in range(args.warmup):
        km.aa_step(None, info=False)
    st0 = km.state_export()
    km.assign_timing()                         # drop warm-up timings
    km.update_timing()
    n_assign0 = st0["n_assign"]
    L0 = km.launch_count()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            km.aa_step(None, info=False)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches = km.launch_count() - L0
    st1 = km.state_export()
    n_assign = st1["n_assign"] - n_assign0
    a_ms, a_n = km.assign_timing()
    u_ms, u_n = km.update_timing()
    ms_max = max_over_ranks(ms, world)
    passes_done = args.steps if not st1["done"] else None
    value = cfg.N * cfg.K * n_assign / (ms_max / 1e3)

    # e2e: host inputs, H2D of the shard + D2H of the result inside the timed region
    C_host = torch.empty(cfg.K, cfg.d, dtype=torch.float64).pin_memory()
    e2e_steps = args.e2e_steps if args.e2e_steps > 0 else args.steps
    with torch.cuda.stream(stream):                               # one untimed e2e step (copy stream, events)
        km.aa_step_host(X_host, chunks=E2E_CHUNKS, info=False)
    barrier()
    st_e0 = km.state_export()["n_assign"]
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tmpC = torch.empty(cfg.K, cfg.d, dtype=torch.float64, device="cuda")
    lib = aakm.lib()
    with torch.cuda.stream(stream):
        for _ in range(e2e_steps):
            # H2D of the step's inputs streamed in row chunks under the assignment, then
            # the rest of one Algorithm 1 pass (C ABI kmeans_aa_step_host)
            km.aa_step_host(X_host, chunks=E2E_CHUNKS, info=False)
            lib.kmeans_get_centroids(km.h, aakm._ptr(tmpC), None)
            C_host.copy_(tmpC, non_blocking=True)                 # D2H of the result C^{t+1}
    e1.record(stream)
    barrier()
    e_ms = e0.elapsed_time(e1)
    wall = time.perf_counter() - t0
    e_na = km.state_export()["n_assign"] - st_e0
    e2e_val = cfg.N * cfg.K * e_na / (max_over_ranks(e_ms, world) / 1e3)

    peaks, peak_kind = load_peaks()
    path = km.path
    n_local = hi - lo
    flops = 2.0 * n_local * cfg.K * cfg.d
    avg_ms = a_ms / max(a_n, 1)
    achieved = flops / (avg_ms / 1e3) / 1e12
    if path == "tc":
        # 3xTF32 (fp32-equivalent): TF32 = bf16 x (1.1/2.25) nominal ratio, three MMAs per product
        peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * (1.1 / 2.25) / 3.0
        bound = "tensor"
    elif path == "tc16":
        # 2xFP16 (fp32-equivalent): fp16 dense = bf16 dense, three MMAs per product
        peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) / 3.0
        bound = "tensor"
    else:
        peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        bound = "alu"
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"{args.config}_{path}_assign_bytes")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f32-exact contraction (2xFP16 / 3xTF32 split + fp64 near-tie refine), f64 state",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: Algorithm 1 passes (m0={cfg.m0}, dynamic m)", "N": cfg.N, "d": cfg.d,
                   "K": cfg.K, "parallelism": f"dp{world}", "assign_path": path,
                   "l2": f"inputs larger than L2 (X shard {n_local * cfg.d * 4 / 1e9:.2f} GB > 126 MB)"},
        "passes": args.steps, "assign_passes": n_assign, "converged_in_window": passes_done is None,
        "iterations_per_s": args.steps / (ms_max / 1e3),
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": n_local * cfg.d * 4,
                "d2h_bytes_per_step": cfg.K * cfg.d * 8, "steps": e2e_steps, "wall_s": wall,
                "h2d": f"pinned host -> device in {E2E_CHUNKS} row chunks overlapping the assignment"},
        "gpu_launches": launches,
        "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                     "kernel": f"assign_{path}", "avg_launch_ms": avg_ms, "launches": a_n},
        "clocks": clk.summary(),
    }
    if u_n:
        u_avg = u_ms / u_n
        ubytes = n_local * cfg.d * 4.0 + n_local * 4.0        # X once + the labels
        line["update_roofline"] = {"bound": "hbm", "achieved": ubytes / (u_avg / 1e3) / 1e9,
                                   "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                   "frac": ubytes / (u_avg / 1e3) / 1e9 / peaks["hbm_gbs"],
                                   # the peak is a copy (read + write); the update is a read stream
                                   # (X once + the labels), which can run slightly above it (a torch
                                   # fp32 sum over the same X measured 6.35 TB/s on this pool)
                                   "peak_kind": "copy (read+write), MEASURED_PEAKS.json",
                                   "kernel": "update (label sort + segmented sums; E from the sums by k_energy_x)",
                                   "avg_ms": u_avg, "launches": u_n}
    km.close()
    if args.ttc_config != "none":
        line["time_to_converge"] = time_to_converge(args.ttc_config, rank, world, barrier)
    if args.seed_config != "none" and world == 1:      # the multi-rank seeding exchange is untested on hardware
        line["seed_pp"] = seed_pp_bench(args.seed_config, rank, world, barrier, peaks)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(X, C0, args.config)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
