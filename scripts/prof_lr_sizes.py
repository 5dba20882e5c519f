"""gpu_list_rank time per call (device-resident int32 succ) for several list
sizes.  HB_PROBE_TRIM=1 returns the allocator pool to the driver between
sizes (does a size's time depend on what ran before it?)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1303_2171_b200.datasets import device_gen_list
from paper_1303_2171_b200 import _lib
from paper_1303_2171_b200.kernels_irregular import gpu_list_rank

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for lg in [int(a) for a in sys.argv[1:]] or [24, 25, 26, 27, 28]:
    n = 1 << lg
    succ, head = device_gen_list(n, 42)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    for _ in range(2):
        gpu_list_rank(succ, head, out=out)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        gpu_list_rank(succ, head, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"n=2^{lg}: {ms:8.3f} ms  {n / ms / 1e6:8.1f} Gnodes/s")
    del succ, out
    torch.cuda.empty_cache()
    if os.environ.get("HB_PROBE_TRIM"):
        _lib.call("hb_trim")
