"""Oracle: work-shared histogram (reference kernels_regular.py:126-169).
Test infrastructure / CPU baseline."""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def check_domain(data: np.ndarray, bins: int) -> None:
    """kernels_regular.py:134-138."""
    if bins < 1:
        raise ValueError("bin_count must be >= 1")
    if data.size and (data.min() < 0 or data.max() >= bins):
        raise ValueError("element outside bin domain")


def side_counts(part: np.ndarray, bins: int, workers: int) -> np.ndarray:
    """kernels_regular.py:149-154: per-worker private histograms, summed."""
    total = np.zeros(bins, dtype=np.int64)
    cuts = np.linspace(0, part.size, workers + 1).astype(int)
    for a, b in zip(cuts[:-1], cuts[1:]):
        total += np.bincount(part[a:b], minlength=bins)
    return total


def hybrid(data: np.ndarray, bins: int, fraction_a: float, workers_a: int = 4, workers_b: int = 4) -> np.ndarray:
    """partition at floor(f·n) (:142-144), both sides concurrently (the
    2-thread pool of worksharing.py:317), merge by summing (:156-160)."""
    check_domain(data, bins)
    cut = int(math.floor(fraction_a * data.size))
    with ThreadPoolExecutor(max_workers=2) as pool:
        fa = pool.submit(side_counts, data[:cut], bins, workers_a)
        fb = pool.submit(side_counts, data[cut:], bins, workers_b)
        return fa.result() + fb.result()


def sequential(data, bins: int) -> np.ndarray:
    """Independent per-element loop (reference tests/oracles.py:41-45)."""
    out = np.zeros(bins, dtype=np.int64)
    for v in np.asarray(data).tolist():
        out[v] += 1
    return out
