"""Pinned host -> device copy rate: one copy vs chunks on 2/4 streams vs
chunked on one stream (1 GiB), and D2H the same."""
import time

import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h.fill_(1)


def rate(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return n / best / 1e9


def split(k, h2d=True):
    streams = [torch.cuda.Stream() for _ in range(k)]

    def run():
        c = n // k
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                if h2d:
                    d[i * c:(i + 1) * c].copy_(h[i * c:(i + 1) * c], non_blocking=True)
                else:
                    h[i * c:(i + 1) * c].copy_(d[i * c:(i + 1) * c], non_blocking=True)
    return run


print("H2D one copy  %.1f GB/s" % rate(lambda: d.copy_(h, non_blocking=True)))
for k in (2, 4, 8):
    print(f"H2D {k} streams %.1f GB/s" % rate(split(k)))
print("D2H one copy  %.1f GB/s" % rate(lambda: h.copy_(d, non_blocking=True)))
for k in (2, 4):
    print(f"D2H {k} streams %.1f GB/s" % rate(split(k, False)))
