"""Oracle: splitmix64 streams (reference rng.py:19-67).  Test infrastructure."""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
G = 0x9E3779B97F4A7C15
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB


def step(state: int) -> tuple[int, int]:
    """rng.py:19-25 — advance by γ, output the xor-shift-multiply finaliser."""
    state = (state + G) & M64
    z = state
    z = ((z ^ (z >> 30)) * C1) & M64
    z = ((z ^ (z >> 27)) * C2) & M64
    return state, z ^ (z >> 31)


def draws_bigint(seed: int, n: int) -> list[int]:
    """Sequential big-int stream (rng.py:28-42 `SplitMix64.next_u64`)."""
    out, s = [], seed & M64
    for _ in range(n):
        s, v = step(s)
        out.append(v)
    return out


def draws(seed: int, n: int, first: int = 1) -> np.ndarray:
    """Vectorised closed form, draws first..first+n-1 (rng.py:45-51)."""
    k = np.arange(first, first + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & M64) + k * np.uint64(G)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(C1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(C2)
    return z ^ (z >> np.uint64(31))


def mix_seed(seed: int, salt: int) -> int:
    """rng.py:54-57."""
    return step((seed ^ (salt * C2)) & M64)[1]


def uniform_floats(seed: int, n: int) -> np.ndarray:
    """rng.py:60-62: top 53 bits scaled to [0, 1)."""
    return (draws(seed, n) >> np.uint64(11)).astype(np.float64) * 2.0**-53


def uniform_ints(seed: int, n: int, bound: int) -> np.ndarray:
    """rng.py:65-67."""
    return (draws(seed, n) % np.uint64(bound)).astype(np.int64)
