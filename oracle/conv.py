"""Oracle: clamp-to-edge correlation on row strips (reference
kernels_regular.py:327-414).  Test infrastructure / CPU baseline only."""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def rows(pixels: np.ndarray, weights: np.ndarray, r0: int, r1: int) -> np.ndarray:
    """:359-381: rows [r0, r1); slab of clamped rows ±r, edge-padded columns,
    one weighted plane added per non-zero tap in row-major (dy, dx) order."""
    h, w = pixels.shape
    r = weights.shape[0] // 2
    m = r1 - r0
    if m <= 0:
        return np.zeros((0, w))
    ridx = np.clip(np.arange(r0 - r, r1 + r), 0, h - 1)
    slab = np.pad(pixels[ridx].astype(np.float64), ((0, 0), (r, r)), mode="edge")
    out = np.zeros((m, w))
    for dy in range(2 * r + 1):
        for dx in range(2 * r + 1):
            wt = weights[dy, dx]
            if wt == 0.0:
                continue
            out += wt * slab[dy : dy + m, dx : dx + w]
    return out


def split(height: int, fraction_a: float) -> int:
    """ConvolutionWorkload.partition (:390-392): floor(f·H)."""
    return int(math.floor(fraction_a * height))


def hybrid(pixels: np.ndarray, weights: np.ndarray, fraction_a: float) -> np.ndarray:
    """hybrid_convolve (:408-414): the two strips computed concurrently, vstacked."""
    s = split(pixels.shape[0], fraction_a)
    with ThreadPoolExecutor(max_workers=2) as ex:
        fa = ex.submit(rows, pixels, weights, 0, s)
        fb = ex.submit(rows, pixels, weights, s, pixels.shape[0])
        return np.vstack([fa.result(), fb.result()])
