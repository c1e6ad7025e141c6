"""Host->device bandwidth from pinned memory: one stream vs two streams (e2e bound)."""
import time

import torch

torch.cuda.set_device(0)
n = 309 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    one = n / (time.perf_counter() - t) / 1e9
    t = time.perf_counter()
    half = n // 2
    with torch.cuda.stream(s1):
        d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        d[half:].copy_(h[half:], non_blocking=True)
    torch.cuda.synchronize()
    two = n / (time.perf_counter() - t) / 1e9
    chunk = 1 << 24
    t = time.perf_counter()
    for i in range(0, n, chunk):
        d[i:i + chunk].copy_(h[i:i + chunk], non_blocking=True)
    torch.cuda.synchronize()
    chunked = n / (time.perf_counter() - t) / 1e9
    print(f"H2D GB/s: one copy {one:.1f}, two streams {two:.1f}, 16 MB chunks {chunked:.1f}")
