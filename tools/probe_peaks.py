"""Measure roofline denominators the driver does not record: TF32 / FP32 / FP64
dense matmul (torch/cuBLAS, burst, CUDA events) plus device properties and host
CPU facts. Output: gpurun_out/peaks_probe.json. Run on the GPU box via gpurun."""
import json, os, subprocess, time
import torch

def bench_mm(dtype, n, iters=10, tf32=False):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); a @ b; e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return 2 * n**3 / best / 1e12

out = {}
p = torch.cuda.get_device_properties(0)
out["device"] = {"name": p.name, "sms": p.multi_processor_count, "total_mem": p.total_memory,
                 "l2": getattr(p, "L2_cache_size", None), "cc": [p.major, p.minor]}
out["tf32_tflops"] = bench_mm(torch.float32, 8192, tf32=True)
out["fp32_tflops"] = bench_mm(torch.float32, 8192, tf32=False)
out["fp64_tflops"] = bench_mm(torch.float64, 4096)
out["bf16_tflops"] = bench_mm(torch.bfloat16, 8192)
out["host_cpus"] = os.cpu_count()
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:1500]
except Exception as ex:
    out["lscpu"] = str(ex)
try:
    out["free"] = subprocess.run(["free", "-g"], capture_output=True, text=True).stdout
    out["nvsmi"] = subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout
except Exception as ex:
    out["nvsmi"] = str(ex)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/peaks_probe.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k not in ("lscpu", "nvsmi", "free")}))
