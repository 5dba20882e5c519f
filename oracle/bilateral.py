"""Oracle: LUT bilateral filter on row strips (reference
kernels_regular.py:421-520, workloads.py:381-398).  Test infrastructure /
CPU baseline."""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def lut(radius: int, sigma_s: float, sigma_r: float) -> tuple[np.ndarray, np.ndarray]:
    """:447-458: spatial (2r+1)^2 row-major, range[k] for k = 0..255."""
    if radius < 0:
        raise ValueError("radius must be >= 0")
    if not (sigma_s > 0 and sigma_r > 0):
        raise ValueError("sigmas must be > 0")
    off = np.arange(-radius, radius + 1, dtype=np.float64)
    d2 = off[:, None] ** 2 + off[None, :] ** 2
    spatial = np.exp(-d2 / (2.0 * sigma_s**2)).ravel()
    k = np.arange(256, dtype=np.float64)
    return spatial, np.exp(-(k**2) / (2.0 * sigma_r**2))


def rows(pixels: np.ndarray, spatial: np.ndarray, rng: np.ndarray, radius: int, r0: int, r1: int) -> np.ndarray:
    """:461-486: clamp-to-edge; taps in row-major (dy, dx) order;
    w = spatial·range[|nb-c|]; num += w·nb; den += w; out = num/den (f64)."""
    h, w = pixels.shape
    m = r1 - r0
    if m <= 0:
        return np.zeros((0, w))
    ridx = np.clip(np.arange(r0 - radius, r1 + radius), 0, h - 1)
    slab = np.pad(pixels[ridx].astype(np.int64), ((0, 0), (radius, radius)), mode="edge")
    c = slab[radius : radius + m, radius : radius + w]
    num = np.zeros((m, w))
    den = np.zeros((m, w))
    side = 2 * radius + 1
    for dy in range(side):
        for dx in range(side):
            nb = slab[dy : dy + m, dx : dx + w]
            wt = spatial[dy * side + dx] * rng[np.abs(nb - c)]
            num += wt * nb
            den += wt
    return num / den


def hybrid(pixels, spatial, rng, radius, fraction_a: float) -> np.ndarray:
    """BilateralApplyWorkload (:489-520): strips split at floor(f·H)."""
    h = pixels.shape[0]
    split = int(math.floor(fraction_a * h))
    with ThreadPoolExecutor(max_workers=2) as pool:
        fa = pool.submit(rows, pixels, spatial, rng, radius, 0, split)
        fb = pool.submit(rows, pixels, spatial, rng, radius, split, h)
        return np.vstack([fa.result(), fb.result()])


def direct(pixels: np.ndarray, radius: int, sigma_s: float, sigma_r: float) -> np.ndarray:
    """LUT-free gate (workloads.py:381-398): exp recomputed per tap."""
    h, w = pixels.shape
    ridx = np.clip(np.arange(-radius, h + radius), 0, h - 1)
    slab = np.pad(pixels[ridx].astype(np.float64), ((0, 0), (radius, radius)), mode="edge")
    c = slab[radius : radius + h, radius : radius + w]
    num = np.zeros((h, w))
    den = np.zeros((h, w))
    for dy in range(-radius, radius + 1):
        for dx in range(-radius, radius + 1):
            nb = slab[dy + radius : dy + radius + h, dx + radius : dx + radius + w]
            wt = math.exp(-(dy * dy + dx * dx) / (2.0 * sigma_s**2)) * np.exp(-((nb - c) ** 2) / (2.0 * sigma_r**2))
            num += wt * nb
            den += wt
    return num / den
