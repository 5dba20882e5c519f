"""Where the list-ranking end-to-end step (host succ -> host ranks) spends its time."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1303_2171_b200.datasets import device_gen_list
from paper_1303_2171_b200.kernels_irregular import gpu_list_rank

n = 1 << 28
succ, head = device_gen_list(n, 42, np.int64)
host = torch.empty(n, dtype=torch.int64, pin_memory=True)
host.copy_(succ)
hn = host.numpy()
def t(fn, k=2):
    fn(); b = []
    for _ in range(k):
        torch.cuda.synchronize(); s = time.perf_counter(); fn(); torch.cuda.synchronize(); b.append(time.perf_counter() - s)
    return min(b) * 1e3
print("host int64 -> host ranks   %.1f ms" % t(lambda: gpu_list_rank(hn, head)))
print("device int64 -> device     %.1f ms" % t(lambda: gpu_list_rank(succ, head)))
s32 = succ.to(torch.int32)
print("device int32 -> device     %.1f ms" % t(lambda: gpu_list_rank(s32, head)))
d = torch.empty(n, dtype=torch.int64, device="cuda")
print("H2D 2 GiB pinned            %.1f ms" % t(lambda: d.copy_(host)))
out = np.empty(n, dtype=np.int64)
print("D2H 2 GiB -> pageable (torch) %.1f ms" % t(lambda: out.__setitem__(slice(None), d.cpu().numpy())))
def fresh():
    o = np.empty(n, dtype=np.int64); o[::512] = 0
print("first-touch 2 GiB numpy      %.1f ms" % t(fresh))
