"""Where the sort's pageable end-to-end call spends its time: 2^28 u32 keys
(pageable numpy), results kept as a plain caller keeps them."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1303_2171_b200.kernels_regular import gpu_sort, sample_sort_hybrid
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

n = 1 << 28
keys = np.random.default_rng(1).integers(0, 1 << 32, size=n, dtype=np.uint32)
p = Platform.build(1.0, 3.0)
sh = WorkShare.manual(0.0)
gpu_sort(keys)
kept = []
for name, fn in [("gpu_sort kept", lambda: kept.append(gpu_sort(keys))),
                 ("gpu_sort dropped", lambda: gpu_sort(keys)),
                 ("sample_sort_hybrid kept", lambda: kept.append(sample_sort_hybrid(keys, p, share=sh)))]:
    ts = []
    for _ in range(3):
        a = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    print(f"{name:28s} " + " ".join(f"{t * 1e3:7.1f}" for t in ts) + " ms", flush=True)
pr = cProfile.Profile()
pr.enable()
kept.append(sample_sort_hybrid(keys, p, share=sh))
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
