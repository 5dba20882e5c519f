"""hb_sort (device, u32 keys + u32 payload, uniform random keys) per call at
several sizes, timed like scripts/micro/cub_sort.cu (fresh keys before each
call, CUDA events around the sort alone) — the library comparison in
profiles/micro_cub_sort_r02.txt."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1303_2171_b200.kernels_regular import gpu_sort

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for lg in [int(a) for a in sys.argv[1:]] or [24, 26, 28, 29]:
    n = 1 << lg
    keys = torch.empty(n, dtype=torch.int64, device="cuda")
    k32 = torch.empty(n, dtype=torch.int32, device="cuda")
    pay = torch.empty(n, dtype=torch.int32, device="cuda")
    ts = []
    for r in range(12):
        keys.random_(0, 1 << 32)
        k32.copy_(keys.to(torch.uint32).view(torch.int32))
        torch.arange(n, out=pay, dtype=torch.int32)
        kv = k32.view(torch.uint32)
        torch.cuda.synchronize()
        e0.record()
        gpu_sort(kv, pay, asynchronous=True)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    ms = sum(ts) / len(ts)
    print(f"hb_sort u32+u32 n=2^{lg}: mean {ms:.3f} ms (best {min(ts):.3f}) = {n / ms / 1e6:.1f} Gkeys/s", flush=True)
    del keys, k32, pay
    torch.cuda.empty_cache()
