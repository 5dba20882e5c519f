"""hb_sort on 2^28 u32 keys + u32 payload (the bench shape) and the list-ranking call at 2^28, CUDA events,
mean of 10 calls after 3 — for A/B runs of two library builds (HB200_LIB)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1303_2171_b200.datasets import device_gen_list
from paper_1303_2171_b200.kernels_irregular import gpu_list_rank
from paper_1303_2171_b200.kernels_regular import gpu_sort

n = 1 << 28
g = torch.Generator(device="cuda").manual_seed(1)
src = torch.randint(0, 1 << 31, (n,), device="cuda", dtype=torch.int64, generator=g).to(torch.int32).view(torch.uint32)
keys = torch.empty_like(src)
vals = torch.empty(n, dtype=torch.int32, device="cuda").view(torch.uint32)
idx = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for i in range(13):
    keys.copy_(src)
    vals.copy_(idx)
    e0.record()
    gpu_sort(keys, vals, asynchronous=True)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
k64 = keys.view(torch.int32).long() & 0xFFFFFFFF
ok = bool((k64[1:] >= k64[:-1]).all()) and bool((src.view(torch.int32)[vals.view(torch.int32).long()] == keys.view(torch.int32)).all())
lib = os.environ.get("HB200_LIB", "default").split("/")[-1]
print(f"{lib:22s} sort 2^28 pairs: {sum(ts) / len(ts):.3f} ms  ({n / (sum(ts) / len(ts)) / 1e6:.0f} Mkeys/s) ok={ok}", flush=True)
for name, dt in (("keys-only u32", torch.int32), ("keys-only u64", torch.int64)):
    ks = torch.randint(0, 1 << 62, (n // (2 if dt == torch.int64 else 1),), device="cuda", dtype=torch.int64,
                       generator=g).to(dt)
    kk = torch.empty_like(ks)
    ts = []
    for i in range(8):
        kk.copy_(ks)
        e0.record()
        gpu_sort(kk, None, asynchronous=True)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    print(f"{lib:22s} sort {name} ({kk.numel()} keys): {sum(ts) / len(ts):.3f} ms", flush=True)
succ, head = device_gen_list(n, 42)
r = torch.empty(n, dtype=torch.int64, device="cuda")
ts = []
for i in range(8):
    e0.record()
    gpu_list_rank(succ, head, out=r, asynchronous=True)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
print(f"{lib:22s} list rank 2^28: {sum(ts) / len(ts):.3f} ms", flush=True)
