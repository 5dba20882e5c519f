"""Hot-path input generators, bit-identical to the reference's
(hybridbench/datasets.py:28-106) but built for benchmark scale: the
splitmix64 streams are closed-form per draw index, so they are generated in
vectorised chunks on the host or directly in HBM (rng.device_splitmix).
"""

from __future__ import annotations

import numpy as np

from .rng import GAMMA, MASK64, mix_seed, splitmix64, splitmix64_array, uniform_floats, uniform_ints

LIST_END = -1


def gen_sort_data(n: int, seed: int) -> np.ndarray:
    """datasets.py:28-30: uniform 32-bit keys as int64."""
    return (splitmix64_array(seed, n) >> np.uint64(32)).astype(np.int64)


def gen_hist_data(n: int, seed: int, bins: int = 256) -> np.ndarray:
    """datasets.py:33-34."""
    return uniform_ints(seed, n, bins)


def gen_image(side: int, seed: int) -> np.ndarray:
    """datasets.py:104-106 pixels (uint8, side x side)."""
    return uniform_ints(seed, side * side, 256).astype(np.uint8).reshape(side, side)


def gen_list(n: int, seed: int) -> tuple[np.ndarray, int]:
    """datasets.py:58-63: (succ int64, head) of one list in stable-argsort
    order of the draws."""
    order = np.argsort(splitmix64_array(seed, n), kind="stable").astype(np.int64)
    succ = np.full(n, LIST_END, dtype=np.int64)
    succ[order[:-1]] = order[1:]
    return succ, int(order[0])


def _fin(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def gen_csr(rows: int, cols: int, seed: int, density: float, chunk_rows: int = 1 << 17):
    """datasets.py:37-55, vectorised: returns (row_ptr, col_idx, values) —
    int64, int64, f64 — bit-identical to the reference generator.

    The reference walks one sequential seed stream, one draw per row plus
    one per retry (a row whose 2k+8 column draws hold fewer than k distinct
    values).  Rows are generated in chunks assuming no retry; the first row
    that needs one is redone exactly as the reference does and the stream
    position of every later row shifts by the retries consumed.
    """
    avg = max(1, round(density * cols))
    counts = np.minimum(1 + uniform_ints(mix_seed(seed, 1), rows, max(1, 2 * avg - 1)), cols)
    base = mix_seed(seed, 2) & MASK64
    pieces: list[np.ndarray] = []
    draw_pos = 0  # draws consumed from the row-seed stream so far
    r = 0
    while r < rows:
        r1 = min(rows, r + chunk_rows)
        k = counts[r:r1].astype(np.int64)
        m = 2 * k + 8
        # seeds of rows r..r1-1 if no retry happens in this chunk
        idx = np.arange(draw_pos + 1, draw_pos + 1 + (r1 - r), dtype=np.uint64)
        with np.errstate(over="ignore"):
            seeds = _fin(np.uint64(base) + idx * np.uint64(GAMMA))
        owner = np.repeat(np.arange(r1 - r, dtype=np.int64), m)
        starts = np.zeros(r1 - r, dtype=np.int64)
        np.cumsum(m[:-1], out=starts[1:])
        j = np.arange(owner.size, dtype=np.int64) - starts[owner] + 1
        with np.errstate(over="ignore"):
            vals = (_fin(seeds[owner] + j.astype(np.uint64) * np.uint64(GAMMA)) % np.uint64(cols)).astype(np.int64)
        key = owner * cols + vals
        key.sort()  # sort + adjacent dedupe (np.unique's hash path is far slower)
        if key.size:
            fresh = np.empty(key.size, dtype=bool)
            fresh[0] = True
            np.not_equal(key[1:], key[:-1], out=fresh[1:])
            key = key[fresh]
        urow = key // cols
        ucol = key - urow * cols
        have = np.bincount(urow, minlength=r1 - r)
        short = np.flatnonzero(have < k)
        stop = int(short[0]) if short.size else r1 - r
        # keep the first k distinct columns of each row before `stop`
        first = np.zeros(r1 - r + 1, dtype=np.int64)
        np.cumsum(have, out=first[1:])
        rank_in_row = np.arange(key.size, dtype=np.int64) - first[urow]
        keep = (rank_in_row < k[urow]) & (urow < stop)
        pieces.append(ucol[keep])
        draw_pos += stop
        r += stop
        if stop < r1 - (r - stop):
            # row r needs retries: replay it exactly like the reference
            draw_pos, chosen = _row_with_retries(base, draw_pos, int(counts[r]), cols)
            pieces.append(chosen)
            r += 1
    col_idx = np.concatenate(pieces) if pieces else np.zeros(0, np.int64)
    row_ptr = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    values = 2.0 * uniform_floats(mix_seed(seed, 3), col_idx.size) - 1.0
    return row_ptr, col_idx, values


def _row_with_retries(base: int, draw_pos: int, k: int, cols: int) -> tuple[int, np.ndarray]:
    state = (base + draw_pos * GAMMA) & MASK64
    state, s = splitmix64(state)
    draw_pos += 1
    chosen = np.unique(uniform_ints(s, 2 * k + 8, cols))
    while chosen.size < k:
        state, s = splitmix64(state)
        draw_pos += 1
        chosen = np.unique(np.concatenate([chosen, np.unique(uniform_ints(s, 2 * k + 8, cols))]))
    return draw_pos, chosen[:k]


def device_gen_list(n: int, seed: int, succ_dtype=np.int32):
    """gen_list on the device, bit-identical to the reference (datasets.py:
    58-63): draws 1..n of `seed` (hb_gen_splitmix), stable argsort by an LSD
    radix sort of the 64-bit draws with an index payload (hb_sort), then
    hb_link_order.  Returns (succ CUDA tensor, head)."""
    import torch

    from . import _lib
    from .gpu import current_stream_handle, vp
    from .rng import device_splitmix

    draws = torch.empty(n, dtype=torch.int64, device="cuda")
    device_splitmix(draws, seed, _lib.HB_GEN_RAW)
    order = torch.arange(n, dtype=torch.int32, device="cuda")
    st = current_stream_handle(draws)
    _lib.call("hb_sort", vp(draws.data_ptr()), vp(draws.data_ptr()), _lib.DTYPE_CODES["u8"], vp(order.data_ptr()),
              vp(order.data_ptr()), n, None, _lib.HB_DEVICE_PTRS, st)
    del draws
    tdt = torch.int32 if np.dtype(succ_dtype) == np.int32 else torch.int64
    succ = torch.empty(n, dtype=tdt, device="cuda")
    _lib.call("hb_link_order", vp(order.data_ptr()), n, vp(succ.data_ptr()),
              _lib.DTYPE_CODES["i4" if tdt == torch.int32 else "i8"], _lib.HB_DEVICE_PTRS, st)
    head = int(order[0].item())
    return succ, head
