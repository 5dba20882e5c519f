"""Capped level-1 walk vs where the successor array lands: a junk allocation
of varying size is made before the list is generated (and kept alive)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1303_2171_b200.datasets import device_gen_list
from paper_1303_2171_b200.kernels_irregular import gpu_list_rank

n = 1 << 28
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for junk_gb in (0, 1, 2, 3, 4.5, 6, 8, 0.25, 0.5):
    junk = torch.empty(int(junk_gb * (1 << 30)), dtype=torch.uint8, device="cuda") if junk_gb else None
    succ, head = device_gen_list(n, 42)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    gpu_list_rank(succ, head, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0.record()
        gpu_list_rank(succ, head, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"junk {junk_gb:4} GB: succ at {succ.data_ptr():#x}: " + " ".join(f"{t:.2f}" for t in ts) + " ms", flush=True)
    del succ, out, junk
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
