"""SpMV end to end on pageable inputs (the bench's pageable leg): time per
call at the bench's share, pinned vs pageable, plus a cProfile of one
pageable call."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench

bench.ARGS.e2e_share = "calibrated"
wl = bench.SpmvBench()
wl.setup(0, 1)
wl.e2e_setup()
print("share", wl.share.fraction_a, flush=True)


def timed(k=6):
    wl.e2e_step()
    ts = []
    for _ in range(k):
        a = time.perf_counter()
        wl.e2e_step()
        ts.append(time.perf_counter() - a)
    return np.median(ts) * 1e3


print(f"pinned   {timed():.2f} ms", flush=True)
wl.e2e_pageable()
print(f"pageable {timed():.2f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
wl.e2e_step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
