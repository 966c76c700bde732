"""Pinned host -> device copy bandwidth (the e2e ceiling); runs under gpurun."""
import time

import torch

torch.cuda.set_device(0)
n = 2_621_440_000 // 2
h = torch.empty(n, dtype=torch.int16).pin_memory()
d = torch.empty(n, dtype=torch.int16, device="cuda")
for chunk_mb in (64, 268, 2621):
    c = chunk_mb * 1_000_000 // 2
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for off in range(0, n, c):
            d[off:off + c].copy_(h[off:off + c], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"H2D chunk {chunk_mb} MB: {n * 2 / dt / 1e9:.1f} GB/s")
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
half = n // 2
d[:half].copy_(h[:half], non_blocking=True)
with torch.cuda.stream(s2):
    d[half:].copy_(h[half:], non_blocking=True)
torch.cuda.synchronize()
print(f"H2D two streams: {n * 2 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
