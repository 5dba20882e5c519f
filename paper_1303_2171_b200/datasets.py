"""Hot-path input generators and on-disk formats, bit-identical to the
reference's (hybridbench/datasets.py:28-163) but built for benchmark scale:
the splitmix64 streams are closed-form per draw index, so they are generated
in vectorised chunks on the host or directly in HBM (rng.device_splitmix).

The public generators return the reference's types (CsrMatrix,
LinkedListArr, Image); the *_arrays helpers return the raw numpy arrays.
Kinds outside this framework's hot path (spgemm's own kernel, cc, lbm) are
not generated here (out of scope) — spgemm inputs are plain
CSR matrices and are served by gen_csr.
"""

from __future__ import annotations

from pathlib import Path
from typing import Any

import numpy as np

from .errors import ConfigError, DataIOError
from .rng import GAMMA, MASK64, mix_seed, splitmix64, splitmix64_array, uniform_floats, uniform_ints

LIST_END = -1
UAR_KINDS = ("sort", "hist", "spmv", "spgemm", "conv", "bilat", "lr")


def gen_sort_data(n: int, seed: int) -> np.ndarray:
    """datasets.py:28-30: uniform 32-bit keys as int64."""
    return (splitmix64_array(seed, n) >> np.uint64(32)).astype(np.int64)


def gen_hist_data(n: int, seed: int, bins: int = 256) -> np.ndarray:
    """datasets.py:33-34."""
    return uniform_ints(seed, n, bins)


def image_pixels(side: int, seed: int) -> np.ndarray:
    """datasets.py:104-106 pixels (uint8, side x side)."""
    return uniform_ints(seed, side * side, 256).astype(np.uint8).reshape(side, side)


def gen_image(side: int, seed: int):
    """datasets.py:104-106 → Image."""
    from .kernels_regular import Image

    return Image(image_pixels(side, seed))


def list_arrays(n: int, seed: int) -> tuple[np.ndarray, int]:
    """datasets.py:58-63: (succ int64, head) of one list in stable-argsort
    order of the draws."""
    order = np.argsort(splitmix64_array(seed, n), kind="stable").astype(np.int64)
    succ = np.full(n, LIST_END, dtype=np.int64)
    succ[order[:-1]] = order[1:]
    return succ, int(order[0])


def gen_list(n: int, seed: int):
    """datasets.py:58-63 → LinkedListArr."""
    from .kernels_irregular import LinkedListArr

    succ, head = list_arrays(n, seed)
    return LinkedListArr(succ, head)


def gen_csr(rows: int, cols: int, seed: int, density: float):
    """datasets.py:37-55 → CsrMatrix (see csr_arrays)."""
    from .kernels_irregular import CsrMatrix

    return CsrMatrix(rows, cols, *csr_arrays(rows, cols, seed, density))


def generate_uar(kind: str, size: int, seed: int, **params: Any):
    """datasets.py:109-130 for the hot-path kinds."""
    if size < 1:
        raise ConfigError(f"dataset size must be >= 1, got {size}")
    if kind == "sort":
        return gen_sort_data(size, seed)
    if kind == "hist":
        return gen_hist_data(size, seed, int(params.get("bins", 256)))
    if kind in ("spmv", "spgemm"):
        return gen_csr(size, size, seed, float(params.get("density", 0.01)))
    if kind == "lr":
        return gen_list(size, seed)
    if kind in ("conv", "bilat"):
        return gen_image(size, seed)
    if kind in ("cc", "lbm"):
        raise ConfigError(f"dataset kind {kind!r} belongs to a workload outside this framework's hot path")
    raise ConfigError(f"unknown dataset kind {kind!r}")


def write_dataset(kind: str, dataset, path: str | Path) -> None:
    """datasets.py:133-153: raw little-endian u32 (sort, hist), MatrixMarket
    (spmv, spgemm), binary PGM (conv, bilat)."""
    if kind in ("sort", "hist"):
        try:
            np.asarray(dataset, dtype=np.uint32).astype("<u4").tofile(path)
        except OSError as exc:
            raise DataIOError(f"cannot write {path}: {exc}") from exc
        return
    if kind in ("spmv", "spgemm"):
        from .kernels_irregular import save_matrix_market

        save_matrix_market(dataset, path)
        return
    if kind in ("conv", "bilat"):
        from .kernels_regular import write_pgm

        write_pgm(dataset, path)
        return
    raise ConfigError(f"dataset kind {kind!r} has no file format; it is generated from config")


def read_raw_u32(path: str | Path) -> np.ndarray:
    """datasets.py:156-163: little-endian u32 file → int64; empty → DataIOError."""
    try:
        data = np.fromfile(path, dtype="<u4")
    except OSError as exc:
        raise DataIOError(f"cannot read {path}: {exc}") from exc
    if data.size == 0:
        raise DataIOError(f"{path}: empty input")
    return data.astype(np.int64)


def _fin(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def csr_arrays(rows: int, cols: int, seed: int, density: float, chunk_rows: int = 1 << 17):
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
    # stable argsort: the ballot ranking (stable by construction)
    _lib.call("hb_sort", vp(draws.data_ptr()), vp(draws.data_ptr()), _lib.DTYPE_CODES["u8"], vp(order.data_ptr()),
              vp(order.data_ptr()), n, None, _lib.HB_DEVICE_PTRS | _lib.HB_SORT_BALLOT, st)
    del draws
    tdt = torch.int32 if np.dtype(succ_dtype) == np.int32 else torch.int64
    succ = torch.empty(n, dtype=tdt, device="cuda")
    _lib.call("hb_link_order", vp(order.data_ptr()), n, vp(succ.data_ptr()),
              _lib.DTYPE_CODES["i4" if tdt == torch.int32 else "i8"], _lib.HB_DEVICE_PTRS, st)
    head = int(order[0].item())
    return succ, head


def device_gen_csr(rows: int, cols: int, seed: int, density: float, index_dtype=np.int32):
    """gen_csr in HBM (hb_gen_csr), bit-identical to the reference
    (datasets.py:37-55) and to `csr_arrays`: a device CsrMatrix with int32
    (default) or int64 row_ptr / col_idx and float64 values."""
    import ctypes

    import torch

    from . import _lib
    from .gpu import current_stream_handle, vp
    from .kernels_irregular import CsrMatrix

    avg = max(1, round(density * cols))
    seeds = [mix_seed(seed, salt) & MASK64 for salt in (1, 2, 3)]
    tdt = torch.int32 if np.dtype(index_dtype) == np.int32 else torch.int64
    code = _lib.DTYPE_CODES["i4" if tdt == torch.int32 else "i8"]
    rp = torch.empty(rows + 1, dtype=torch.int64, device="cuda")
    nnz = ctypes.c_int64(0)
    st = current_stream_handle(rp)
    _lib.call("hb_gen_csr", rows, cols, avg, *seeds, vp(rp.data_ptr()), _lib.DTYPE_CODES["i8"], None, code, None, 0,
              ctypes.byref(nnz), _lib.HB_DEVICE_PTRS, st)
    nnz = nnz.value
    ptr_t = tdt if nnz < 2**31 else torch.int64
    rp = torch.empty(rows + 1, dtype=ptr_t, device="cuda")
    col = torch.empty(nnz, dtype=tdt, device="cuda")
    val = torch.empty(nnz, dtype=torch.float64, device="cuda")
    out = ctypes.c_int64(0)
    _lib.call("hb_gen_csr", rows, cols, avg, *seeds, vp(rp.data_ptr()),
              _lib.DTYPE_CODES["i4" if ptr_t == torch.int32 else "i8"], vp(col.data_ptr()), code, vp(val.data_ptr()),
              nnz, ctypes.byref(out), _lib.HB_DEVICE_PTRS, st)
    return CsrMatrix(rows, cols, rp, col, val)


def device_gen_sort_data(n: int, seed: int, k0: int = 0):
    """gen_sort_data in HBM: uint32 keys (draw >> 32) of draws k0+1..k0+n,
    as an int32 tensor holding the same bits."""
    import torch

    from . import _lib
    from .rng import device_splitmix

    out = torch.empty(n, dtype=torch.int32, device="cuda")
    device_splitmix(out, seed, _lib.HB_GEN_HI32, k0=k0)
    return out


def device_gen_image(side: int, seed: int, k0: int = 0):
    """gen_image pixels in HBM (uint8 side x side, draw & 255)."""
    import torch

    from . import _lib
    from .rng import device_splitmix

    out = torch.empty((side, side), dtype=torch.uint8, device="cuda")
    device_splitmix(out, seed, _lib.HB_GEN_LOW8, k0=k0)
    return out


def device_gen_hist_data(n: int, seed: int, bins: int = 256, k0: int = 0):
    """gen_hist_data in HBM: uint8 for bins <= 256 (draw & 255 when bins is
    256, draw % bins otherwise), int64 above."""
    import torch

    from . import _lib
    from .rng import device_splitmix

    if bins == 256:
        out = torch.empty(n, dtype=torch.uint8, device="cuda")
        device_splitmix(out, seed, _lib.HB_GEN_LOW8, k0=k0)
        return out
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    device_splitmix(out, seed, _lib.HB_GEN_MOD, bound=bins, k0=k0)
    return out if bins > 256 else out.to(torch.uint8)
