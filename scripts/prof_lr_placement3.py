"""Does the library's memory-pool state flip the capped walk between its
fast and slow modes?  Rank a 2^27 list first (its log and pair buffers go
through the pool), then the 2^28 list — with and without hb_trim between."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1303_2171_b200 import _lib
from paper_1303_2171_b200.datasets import device_gen_list
from paper_1303_2171_b200.kernels_irregular import gpu_list_rank

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(succ, head, out, label):
    gpu_list_rank(succ, head, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0.record()
        gpu_list_rank(succ, head, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{label}: " + " ".join(f"{t:.2f}" for t in ts) + " ms", flush=True)


big, hb = device_gen_list(1 << 28, 42)
ob = torch.empty(1 << 28, dtype=torch.int64, device="cuda")
timed(big, hb, ob, "2^28 fresh")
for pre in (25, 26, 27):
    small, hs = device_gen_list(1 << pre, 7)
    os_ = torch.empty(1 << pre, dtype=torch.int64, device="cuda")
    gpu_list_rank(small, hs, out=os_)
    torch.cuda.synchronize()
    timed(big, hb, ob, f"2^28 after a 2^{pre} call")
    _lib.load().hb_trim()
    timed(big, hb, ob, f"2^28 after hb_trim")
    del small, os_
