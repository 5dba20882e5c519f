"""Per-key cost of the LSD sort (u32 keys + u32 payload, 4 passes) when the
working set fits in L2 (2^20..2^23 keys) vs the 2^28 config: is a pass bound
by DRAM or by the SM side?  Feasibility probe for an MSD-then-in-L2 design."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1303_2171_b200 import _lib
from paper_1303_2171_b200.kernels_regular import gpu_sort
from paper_1303_2171_b200.rng import device_splitmix

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for lg in (20, 21, 22, 23, 24, 26, 28):
    n = 1 << lg
    src = torch.empty(n, dtype=torch.int64, device="cuda")
    device_splitmix(src, 42, _lib.HB_GEN_HI32)
    keys0 = src.to(torch.int32)  # bit pattern of the high 32 bits
    keys0 = keys0.view(torch.uint32) if hasattr(torch, "uint32") else keys0
    idx0 = torch.arange(n, dtype=torch.int32, device="cuda")
    reps = max(3, (1 << 26) // n)
    bufs = [(keys0.clone(), idx0.clone()) for _ in range(2)]
    for k, v in bufs:
        gpu_sort(k, v, asynchronous=True)
    torch.cuda.synchronize()
    tot = 0.0
    for r in range(reps):
        k, v = bufs[r % 2]
        k.copy_(keys0)
        v.copy_(idx0)
        e0.record()
        gpu_sort(k, v, asynchronous=True)
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    ms = tot / reps
    print(f"n=2^{lg}: {ms * 1e3:9.1f} us/sort  {n / ms / 1e6:7.2f} Gkeys/s  {n * 68 / ms / 1e6:6.0f} GB/s (68 B/key)")
