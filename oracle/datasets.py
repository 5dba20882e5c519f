"""Oracle: the hot-path input generators (reference datasets.py:28-106).
Test infrastructure; also builds the bench's host-side inputs for the CPU
baseline leg."""

from __future__ import annotations

import numpy as np

from .rng import draws, mix_seed, step, uniform_floats, uniform_ints


def sort_keys(n: int, seed: int) -> np.ndarray:
    """datasets.py:28-30: high 32 bits of draws 1..n (int64)."""
    return (draws(seed, n) >> np.uint64(32)).astype(np.int64)


def hist_values(n: int, seed: int, bins: int = 256) -> np.ndarray:
    """datasets.py:33-34: draw % bins (int64)."""
    return uniform_ints(seed, n, bins)


def image(side: int, seed: int) -> np.ndarray:
    """datasets.py:104-106: low byte of draws, side x side uint8."""
    return uniform_ints(seed, side * side, 256).astype(np.uint8).reshape(side, side)


def linked_list(n: int, seed: int) -> tuple[np.ndarray, int]:
    """datasets.py:58-63: nodes chained in stable-argsort order of the draws."""
    order = np.argsort(draws(seed, n), kind="stable").astype(np.int64)
    succ = np.full(n, -1, dtype=np.int64)
    succ[order[:-1]] = order[1:]
    return succ, int(order[0])


def csr(rows: int, cols: int, seed: int, density: float):
    """datasets.py:37-55, row by row exactly as the reference walks its
    sequential per-row seed stream (with the retry loop).  Returns
    (row_ptr int64, col_idx int64, values f64)."""
    avg = max(1, round(density * cols))
    counts = np.minimum(1 + uniform_ints(mix_seed(seed, 1), rows, max(1, 2 * avg - 1)), cols)
    state = mix_seed(seed, 2) & ((1 << 64) - 1)
    chunks = []
    for k in counts.tolist():
        state, s = step(state)
        picked = np.unique(uniform_ints(s, 2 * k + 8, cols))
        while picked.size < k:
            state, s = step(state)
            picked = np.unique(np.concatenate([picked, np.unique(uniform_ints(s, 2 * k + 8, cols))]))
        chunks.append(picked[:k])
    col_idx = np.concatenate(chunks) if chunks else np.zeros(0, np.int64)
    row_ptr = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    values = 2.0 * uniform_floats(mix_seed(seed, 3), col_idx.size) - 1.0
    return row_ptr, col_idx.astype(np.int64), values
