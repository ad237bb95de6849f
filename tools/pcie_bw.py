"""Host<->device copy bandwidth, pageable vs pinned, at the e2e sizes (12.8 MB)."""
import time
import torch
n = 12_800_000 // 8
d = torch.empty(n, dtype=torch.float64, device="cuda")
for pinned in (False, True):
    h = torch.empty(n, dtype=torch.float64, pin_memory=pinned)
    h.fill_(1.0)
    for direction in ("h2d", "d2h"):
        for _ in range(3):
            (d.copy_(h) if direction == "h2d" else h.copy_(d)); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            (d.copy_(h) if direction == "h2d" else h.copy_(d))
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 20
        print(f"{'pinned ' if pinned else 'pageable'} {direction}: {dt * 1e3:.3f} ms, {h.numel() * 8 / dt / 1e9:.1f} GB/s")
