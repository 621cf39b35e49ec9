"""Pinned host <-> device copy bandwidth (the e2e floor)."""
import torch, time
for mb in (32, 84):
    n = mb * 1024 * 1024 // 8
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    h2d = mb * 10 / (time.perf_counter() - t) / 1024
    t = time.perf_counter()
    for _ in range(10):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    d2h = mb * 10 / (time.perf_counter() - t) / 1024
    print(f"{mb} MB: H2D {h2d:.1f} GB/s, D2H {d2h:.1f} GB/s")
