"""Oracle: the reference's hybrid sample sort (kernels_regular.py:175-321).
Test infrastructure / CPU baseline (`kind: port`)."""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

FANOUT = 64  # SORT_FANOUT, kernels_regular.py:175
CELLS = 256  # SORT_HIST_CELLS, :176
MAX_DEPTH = 8  # SORT_MAX_DEPTH, :177


def insertion_sort_inplace(a: np.ndarray) -> None:
    """:180-187 (DeviceB leaves)."""
    for i in range(1, a.size):
        v = a[i]
        j = i - 1
        while j >= 0 and a[j] > v:
            a[j + 1] = a[j]
            j -= 1
        a[j + 1] = v


def cell_of(chunk: np.ndarray, lo, hi) -> np.ndarray:
    """:201-204: f64 cell index, truncated then clipped to [0, 255]."""
    scale = CELLS / (float(hi) - float(lo))
    return np.clip(((chunk - float(lo)) * scale).astype(np.int64), 0, CELLS - 1)


def splitters_from(counts: np.ndarray, n: int, lo, hi) -> np.ndarray:
    """:190-198: 63 equal-mass cuts of the cell histogram, as unique values."""
    cum = np.cumsum(counts)
    targets = np.arange(1, FANOUT) * (n / FANOUT)
    cells = np.searchsorted(cum, targets, side="left")
    return np.unique(float(lo) + (cells + 1) * ((float(hi) - float(lo)) / CELLS))


def bins_of(chunk: np.ndarray, splitters: np.ndarray) -> list[np.ndarray]:
    """:207-213: stable distribution into len(splitters)+1 value bins."""
    ids = np.searchsorted(splitters, chunk, side="right")
    arranged = chunk[np.argsort(ids, kind="stable")]
    sizes = np.bincount(ids, minlength=splitters.size + 1)
    edges = np.concatenate([[0], np.cumsum(sizes)])
    return [arranged[edges[i] : edges[i + 1]] for i in range(sizes.size)]


def sort_bin(chunk: np.ndarray, leaf: int, depth: int, insertion: bool) -> np.ndarray:
    """:216-236 recursive splitter sort."""
    if chunk.size <= 1:
        return chunk
    if chunk.size <= leaf:
        if insertion:
            out = chunk.copy()
            insertion_sort_inplace(out)
            return out
        return np.sort(chunk, kind="quicksort")
    if depth >= MAX_DEPTH:
        return np.sort(chunk, kind="quicksort")
    lo, hi = chunk.min(), chunk.max()
    if lo == hi:
        return chunk
    spl = splitters_from(np.bincount(cell_of(chunk, lo, hi), minlength=CELLS), chunk.size, lo, hi)
    if spl.size == 0:
        return np.sort(chunk, kind="quicksort")
    return np.concatenate([sort_bin(b, leaf, depth + 1, insertion) for b in bins_of(chunk, spl)])


def plan(arr: np.ndarray, fraction: float):
    """The binning + smallest-bins-first cut of :264-292.  Returns
    (bins, on_a) or None for the early-return cases handled by the caller."""
    n = arr.size
    lo, hi = arr.min(), arr.max()
    if lo == hi:
        return None
    split = int(math.floor(fraction * n))
    cells = cell_of(arr, lo, hi)
    counts = np.bincount(cells[:split], minlength=CELLS) + np.bincount(cells[split:], minlength=CELLS)
    spl = splitters_from(counts, n, lo, hi)
    if spl.size == 0:
        return None
    bins = bins_of(arr, spl)
    sizes = np.array([b.size for b in bins])
    asc = np.argsort(sizes, kind="stable")
    prefix = np.concatenate([[0.0], np.cumsum(sizes[asc])])
    if fraction <= 0.0:
        cut = 0
    elif fraction >= 1.0:
        cut = len(bins)
    else:
        cut = int(np.argmin(np.maximum(prefix / fraction, (n - prefix) / (1.0 - fraction))))
    on_a = np.zeros(len(bins), dtype=bool)
    on_a[asc[:cut]] = True
    return bins, on_a


def sample_sort_hybrid(data, fraction: float, leaf_a: int = 2048, leaf_b: int = 32):
    """:239-310 → (sorted, work_a, work_b)."""
    if not leaf_a >= leaf_b >= 2:
        raise ValueError("need leaf_a >= leaf_b >= 2")
    arr = np.asarray(data)
    n = arr.size
    if n <= 1:
        return arr.copy(), float(n), 0.0
    if n <= leaf_a:
        return np.sort(arr, kind="quicksort"), float(n), 0.0
    p = plan(arr, fraction)
    if p is None:
        lo_eq = arr.min() == arr.max()
        return (arr.copy() if lo_eq else np.sort(arr, kind="quicksort")), float(n), 0.0
    bins, on_a = p
    out: list[np.ndarray] = [np.empty(0, dtype=arr.dtype)] * len(bins)

    def side(is_a: bool) -> None:
        for i, b in enumerate(bins):
            if on_a[i] == is_a:
                out[i] = sort_bin(b, leaf_a if is_a else leaf_b, 1, insertion=not is_a)

    with ThreadPoolExecutor(max_workers=2) as pool:
        fa, fb = pool.submit(side, True), pool.submit(side, False)
        fa.result(), fb.result()
    work_a = float(sum(b.size for b, a in zip(bins, on_a) if a))
    return np.concatenate(out), work_a, float(n) - work_a


def check_stable_payload(keys_in: np.ndarray, keys_out: np.ndarray, payload_out: np.ndarray) -> bool:
    """O(n) proof that payload_out is the stable argsort of keys_in, given
    payload_in = arange(n): it is a permutation, it gathers the sorted keys,
    and within runs of equal keys it is increasing."""
    n = keys_in.size
    p = payload_out.astype(np.int64)
    if p.size != n or (n and (p.min() < 0 or p.max() >= n)):
        return False
    if not np.array_equal(np.bincount(p, minlength=n), np.ones(n, dtype=np.int64)):
        return False
    if not np.array_equal(keys_in[p], keys_out):
        return False
    if n < 2:
        return True
    return bool(np.all((np.diff(keys_out.astype(np.int64)) > 0) | (np.diff(p) > 0)))
