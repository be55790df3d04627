"""Host<->device copy rates for pinned 8 GB buffers (1 and 2 streams): the
floor under bench.py's e2e (H2D of T, D2H of X and E)."""
import time

import torch

n = 1 << 30  # doubles (8 GiB)
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for rep in range(2):
    t = timed(lambda: d.copy_(h, non_blocking=True))
    print(f"H2D 1 stream: {8 * n / t / 1e9:.1f} GB/s")
    t = timed(lambda: h.copy_(d, non_blocking=True))
    print(f"D2H 1 stream: {8 * n / t / 1e9:.1f} GB/s")

    def two():
        with torch.cuda.stream(s1):
            h[: n // 2].copy_(d[: n // 2], non_blocking=True)
        with torch.cuda.stream(s2):
            h[n // 2:].copy_(d[n // 2:], non_blocking=True)
    t = timed(two)
    print(f"D2H 2 streams: {8 * n / t / 1e9:.1f} GB/s")

    def both():
        with torch.cuda.stream(s1):
            h.copy_(d, non_blocking=True)
        with torch.cuda.stream(s2):
            d2 = d  # same device buffer read; H2D into a second region would need 16 GB
            h2[: n // 2].copy_(d2[: n // 2], non_blocking=True)
    t = timed(lambda: d.copy_(h, non_blocking=True))
