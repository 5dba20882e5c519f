"""Oracle: nnz-sorted CSR SpMV with row split (reference
kernels_irregular.py:153-257).  Test infrastructure / CPU baseline."""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np


def permute_rows(row_ptr, col_idx, values, perm):
    """:171-183: gather rows in `perm` order."""
    rows = row_ptr.size - 1
    nnz_of = np.diff(row_ptr)
    counts = nnz_of[perm]
    new_ptr = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(counts, out=new_ptr[1:])
    nnz = int(col_idx.size)
    if nnz:
        src = np.arange(nnz, dtype=np.int64) - np.repeat(new_ptr[:-1], counts) + np.repeat(row_ptr[perm], counts)
    else:
        src = np.zeros(0, dtype=np.int64)
    return new_ptr, col_idx[src], values[src]


def preprocess(row_ptr, col_idx, values, thr_a: float, thr_b: float, fraction_a: float | None):
    """:186-203 → (perm, permuted (ptr, col, val), split_row)."""
    perm = np.argsort(np.diff(row_ptr), kind="stable")
    p_ptr, p_col, p_val = permute_rows(row_ptr, col_idx, values, perm)
    cum = np.concatenate([[0], np.cumsum(np.diff(p_ptr))]).astype(np.float64)
    total = cum[-1]
    if fraction_a is not None:
        split = int(np.searchsorted(cum, fraction_a * total, side="left"))
    else:
        split = int(np.argmin(np.maximum(cum / thr_a, (total - cum) / thr_b)))
    return perm, (p_ptr, p_col, p_val), split


def workload_split(row_ptr_perm, fraction_a: float) -> int:
    """SpmvWorkload.partition (:243-245): searchsorted on the f64 nnz prefix."""
    cum = np.concatenate([[0], np.cumsum(np.diff(row_ptr_perm))]).astype(float)
    return int(np.searchsorted(cum, fraction_a * cum[-1], side="left"))


def range_matvec(ptr, col, val, x, r0: int, r1: int) -> np.ndarray:
    """:206-211: f64 products, then per-row left-to-right sums (bincount)."""
    lo, hi = ptr[r0], ptr[r1]
    owner = np.repeat(np.arange(r1 - r0), np.diff(ptr[r0 : r1 + 1]))
    return np.bincount(owner, weights=val[lo:hi] * x[col[lo:hi]], minlength=r1 - r0)


def hybrid(perm, permuted, split: int, x) -> np.ndarray:
    """:214-227: two row ranges concurrently, concat, inverse-permute."""
    ptr, col, val = permuted
    x = np.asarray(x, dtype=np.float64)
    rows = ptr.size - 1
    with ThreadPoolExecutor(max_workers=2) as pool:
        fa = pool.submit(range_matvec, ptr, col, val, x, 0, split)
        fb = pool.submit(range_matvec, ptr, col, val, x, split, rows)
        y_perm = np.concatenate([fa.result(), fb.result()])
    y = np.empty_like(y_perm)
    y[perm] = y_perm
    return y


def sequential_rows(ptr, col, val, x) -> np.ndarray:
    """Per-row sequential fp64 sum without FMA — the arithmetic the reference's
    bincount performs (used to pin bit-exactness independently of numpy)."""
    rows = ptr.size - 1
    y = np.zeros(rows)
    for r in range(rows):
        acc = 0.0
        for k in range(int(ptr[r]), int(ptr[r + 1])):
            acc = acc + float(val[k]) * float(x[int(col[k])])
        y[r] = acc
    return y
