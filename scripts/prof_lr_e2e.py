"""Where the list-ranking end-to-end call (host int64 succ → ranks) spends its time."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1303_2171_b200.datasets import device_gen_list  # noqa: E402
from paper_1303_2171_b200.kernels_irregular import gpu_list_rank  # noqa: E402

n = 1 << 28
succ, head = device_gen_list(n, 42)
s64 = succ.to(torch.int64)
host = torch.empty(n, dtype=torch.int64, pin_memory=True)
host.copy_(s64)
hnp = host.numpy()


def t(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3, float(np.mean(ts)) * 1e3


out = torch.empty(n, dtype=torch.int64, device="cuda")
print("device int32 succ   %.2f / %.2f ms" % t(lambda: gpu_list_rank(succ, head, out=out)))
print("device int64 succ   %.2f / %.2f ms" % t(lambda: gpu_list_rank(s64, head, out=out)))
print("host pinned int64   %.2f / %.2f ms" % t(lambda: gpu_list_rank(hnp, head)))
r = None
def keep():
    global r
    r = None
    r = gpu_list_rank(hnp, head)
print("host, drop result   %.2f / %.2f ms" % t(keep))
print("H2D 2 GiB           %.2f / %.2f ms" % t(lambda: s64.copy_(host, non_blocking=True)))
print("D2H 2 GiB           %.2f / %.2f ms" % t(lambda: host.copy_(s64, non_blocking=True)))
