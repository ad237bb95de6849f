"""Pinned H2D bandwidth with 1, 2 and 4 concurrent streams (copy-engine parallelism)."""
import time
import torch
n = 25_600_000 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True); h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    step = n // ns
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for k in range(10):
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 10
    print(f"{ns} streams: {n * 8 / dt / 1e9:.1f} GB/s")
