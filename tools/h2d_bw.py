import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        per = n // streams
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * per:(i + 1) * per].copy_(h[i * per:(i + 1) * per], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(streams, "streams:", 4 * n / dt / 1e9, "GB/s")
