"""Is the capped level-1 walk's speed a function of where its buffers land?
The same 2^28-node list ranked repeatedly while a spacer allocation of a
different size shifts the stream-ordered pool's placement between calls."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1303_2171_b200 import _lib
from paper_1303_2171_b200.datasets import device_gen_list
from paper_1303_2171_b200.kernels_irregular import gpu_list_rank

n = 1 << 28
succ, head = device_gen_list(n, 42)
out = torch.empty(n, dtype=torch.int64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for spacer_mb in (0, 0, 0, 64, 128, 256, 512, 1024, 3, 7, 2048):
    lib = _lib.load()
    lib.hb_trim()
    sp = torch.empty(spacer_mb << 20, dtype=torch.uint8, device="cuda") if spacer_mb else None
    gpu_list_rank(succ, head, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0.record()
        gpu_list_rank(succ, head, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"spacer {spacer_mb:5d} MB: " + " ".join(f"{t:.2f}" for t in ts) + " ms", flush=True)
    del sp
