"""Irregular hot-path kernels behind the reference's own entry points
(hybridbench/kernels_irregular.py): CSR SpMV (+ MatrixMarket I/O) and list
ranking.

Same names, signatures and error behaviour as the reference.  DeviceA (host
share) runs numpy on the host cores; DeviceB (GPU share) is one libhb200
call.  Matrices may hold numpy arrays (host; staged per call) or CUDA
tensors (device-resident; `CsrMatrix.to_device()`), in which case the whole
DeviceB path stays in HBM.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from pathlib import Path
from typing import Any, Sequence

import numpy as np

from . import _lib, sharding
from .errors import DataIOError, StructuralError
from .gpu import buf, current_stream_handle, host_empty, inherit_device, is_device_array, require_gpu, to_host, vp
from .platform import Device, DeviceId, Platform
from .worksharing import WorkShare, formula_share, run_workshared

LIST_END = -1

# --------------------------------------------------------------------------
# CSR matrices (kernels_irregular.py:36-98)


def _index_code(a: Any) -> int:
    dt = a.dtype if not is_device_array(a) else np.dtype(str(a.dtype).replace("torch.", ""))
    if dt == np.int32:
        return _lib.DTYPE_CODES["i4"]
    if dt == np.int64:
        return _lib.DTYPE_CODES["i8"]
    raise TypeError(f"index arrays must be int32 or int64, got {dt}")


@dataclass(frozen=True)
class CsrMatrix:
    """CSR with the reference invariants (row_ptr 0..nnz non-decreasing,
    columns in range and strictly increasing per row), checked on
    construction — with numpy for host arrays, with hb_csr_validate for CUDA
    tensors."""

    rows: int
    cols: int
    row_ptr: Any
    col_idx: Any
    values: Any

    def __post_init__(self) -> None:
        if self.rows < 1 or self.cols < 1:
            raise StructuralError("matrix dimensions must be positive")
        rp, ci, v = self.row_ptr, self.col_idx, self.values
        if tuple(rp.shape) != (self.rows + 1,):
            raise StructuralError("row_ptr must run from 0 to nnz with rows+1 entries")
        if tuple(ci.shape) != tuple(v.shape):
            raise StructuralError("col_idx and values must have equal length")
        if is_device_array(rp):
            self._validate_device()
            return
        if rp[0] != 0 or rp[-1] != ci.size:
            raise StructuralError("row_ptr must run from 0 to nnz with rows+1 entries")
        if np.any(np.diff(rp) < 0):
            raise StructuralError("row_ptr must be non-decreasing")
        if ci.size and (ci.min() < 0 or ci.max() >= self.cols):
            raise StructuralError("column index out of range")
        if ci.size:
            owner = np.repeat(np.arange(self.rows), np.diff(rp))
            same = owner[1:] == owner[:-1]
            if np.any(np.diff(ci)[same] <= 0):
                raise StructuralError("column indices must be strictly increasing per row")

    def _validate_device(self) -> None:
        import ctypes

        require_gpu()
        out = ctypes.c_uint32(0)
        _lib.call(
            "hb_csr_validate", vp(self.row_ptr.data_ptr()), _index_code(self.row_ptr),
            vp(self.col_idx.data_ptr()), _index_code(self.col_idx), self.rows, self.nnz, self.cols,
            ctypes.byref(out), _lib.HB_DEVICE_PTRS, current_stream_handle(self.row_ptr),
        )
        f = out.value
        if f & 1:
            raise StructuralError("row_ptr must run from 0 to nnz with rows+1 entries")
        if f & 2:
            raise StructuralError("row_ptr must be non-decreasing")
        if f & 4:
            raise StructuralError("column index out of range")
        if f & 8:
            raise StructuralError("column indices must be strictly increasing per row")

    @property
    def on_device(self) -> bool:
        return is_device_array(self.row_ptr)

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel() if self.on_device else self.col_idx.size)

    @property
    def row_nnz(self) -> np.ndarray:
        return np.diff(to_host(self.row_ptr))

    def to_dense(self) -> np.ndarray:
        rp, ci, v = to_host(self.row_ptr), to_host(self.col_idx), to_host(self.values)
        dense = np.zeros((self.rows, self.cols))
        dense[np.repeat(np.arange(self.rows), np.diff(rp)), ci] = v
        return dense

    def to_device(self, index_dtype: Any = np.int32) -> "CsrMatrix":
        """Device-resident copy (int32 column indices by default: 12 B/nnz)."""
        import torch

        require_gpu()
        tdt = torch.int32 if np.dtype(index_dtype) == np.int32 else torch.int64
        pdt = torch.int32 if self.nnz < 2**31 and tdt == torch.int32 else torch.int64
        rp = torch.from_numpy(np.ascontiguousarray(to_host(self.row_ptr))).to("cuda", pdt)
        ci = torch.from_numpy(np.ascontiguousarray(to_host(self.col_idx))).to("cuda", tdt)
        v = torch.from_numpy(np.ascontiguousarray(to_host(self.values), dtype=np.float64)).to("cuda")
        return CsrMatrix(self.rows, self.cols, rp, ci, v)

    def to_host(self) -> "CsrMatrix":
        if not self.on_device:
            return self
        return CsrMatrix(self.rows, self.cols, to_host(self.row_ptr).astype(np.int64),
                         to_host(self.col_idx).astype(np.int64), to_host(self.values))

    @classmethod
    def from_coo(cls, rows: int, cols: int, r, c, v) -> "CsrMatrix":
        """Coordinate triples; duplicates summed (kernels_irregular.py:76-93)."""
        r = np.asarray(r, dtype=np.int64)
        c = np.asarray(c, dtype=np.int64)
        v = np.asarray(v, dtype=np.float64)
        order = np.lexsort((c, r))
        r, c, v = r[order], c[order], v[order]
        if r.size:
            first = np.ones(r.size, dtype=bool)
            first[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
            starts = np.flatnonzero(first)
            v = np.add.reduceat(v, starts)
            r, c = r[starts], c[starts]
        row_ptr = np.zeros(rows + 1, dtype=np.int64)
        np.cumsum(np.bincount(r, minlength=rows), out=row_ptr[1:])
        return cls(rows, cols, row_ptr, c, v)

    @classmethod
    def identity(cls, n: int) -> "CsrMatrix":
        idx = np.arange(n, dtype=np.int64)
        return cls(n, n, np.arange(n + 1, dtype=np.int64), idx, np.ones(n))


# --------------------------------------------------------------------------
# SpMV (kernels_irregular.py:149-257)


def load_matrix_market(path: str | Path) -> CsrMatrix:
    """kernels_irregular.py:101-134: coordinate real MatrixMarket, general or
    symmetric (off-diagonal entries mirrored), duplicates summed (from_coo);
    malformed input → DataIOError."""
    try:
        with open(path, "r", encoding="ascii") as fh:
            banner = fh.readline().strip().lower().split()
            if banner[:4] != ["%%matrixmarket", "matrix", "coordinate", "real"]:
                raise DataIOError(f"{path}: only coordinate real MatrixMarket is supported")
            symmetry = banner[4] if len(banner) > 4 else "general"
            if symmetry not in ("general", "symmetric"):
                raise DataIOError(f"{path}: unsupported symmetry {symmetry!r}")
            line = fh.readline()
            while line.startswith("%"):
                line = fh.readline()
            rows, cols, nnz = (int(t) for t in line.split())
            body = fh.read().split()
    except DataIOError:
        raise
    except (OSError, ValueError, IndexError) as exc:
        raise DataIOError(f"cannot read MatrixMarket file {path}: {exc}") from exc
    if len(body) % 3 or len(body) // 3 != nnz:
        raise DataIOError(f"{path}: expected {nnz} entries, found {len(body) / 3:g}")
    try:
        trip = np.array(body, dtype=np.float64).reshape(-1, 3) if nnz else np.zeros((0, 3))
    except ValueError as exc:
        raise DataIOError(f"cannot read MatrixMarket file {path}: {exc}") from exc
    r = trip[:, 0].astype(np.int64) - 1
    c = trip[:, 1].astype(np.int64) - 1
    v = trip[:, 2]
    if symmetry == "symmetric":
        mirror = r != c
        r, c, v = np.concatenate([r, c[mirror]]), np.concatenate([c, r[mirror]]), np.concatenate([v, v[mirror]])
    try:
        return CsrMatrix.from_coo(rows, cols, r, c, v)
    except StructuralError as exc:
        raise DataIOError(f"{path}: {exc}") from exc


def save_matrix_market(m: CsrMatrix, path: str | Path) -> None:
    """kernels_irregular.py:137-146: general coordinate file, 1-based
    indices, values written with repr (round-trip exact)."""
    m = m.to_host() if m.on_device else m
    rows_of = np.repeat(np.arange(m.rows), m.row_nnz)
    try:
        with open(path, "w", encoding="ascii") as fh:
            fh.write(f"%%MatrixMarket matrix coordinate real general\n{m.rows} {m.cols} {m.nnz}\n")
            fh.writelines(f"{r + 1} {c + 1} {v!r}\n" for r, c, v in
                          zip(rows_of.tolist(), np.asarray(m.col_idx).tolist(), np.asarray(m.values, dtype=np.float64).tolist()))
    except OSError as exc:
        raise DataIOError(f"cannot write MatrixMarket file {path}: {exc}") from exc


@dataclass(frozen=True)
class SpmvPrep:
    """Rows stably sorted by ascending nnz; rows before split_row (sparse)
    belong to DeviceA, the dense remainder to DeviceB (:153-168)."""

    permuted: CsrMatrix
    perm: Any
    split_row: int
    workers_a: int = 1  # host threads for the DeviceA rows (extension; the platform's DeviceA workers)

    def __post_init__(self) -> None:
        perm = np.asarray(to_host(self.perm), dtype=np.int64)
        n = self.permuted.rows
        if perm.shape != (n,) or not np.array_equal(np.sort(perm), np.arange(n)):
            raise StructuralError("perm must be a permutation of the row indices")
        if np.any(np.diff(self.permuted.row_nnz) < 0):
            raise StructuralError("permuted rows must have non-decreasing nnz")
        if not 0 <= self.split_row <= n:
            raise StructuralError("split_row out of range")


def _permute_rows_host(m: CsrMatrix, perm: np.ndarray) -> CsrMatrix:
    rp = to_host(m.row_ptr).astype(np.int64)
    counts = np.diff(rp)[perm]
    new_ptr = np.zeros(m.rows + 1, dtype=np.int64)
    np.cumsum(counts, out=new_ptr[1:])
    src = (np.arange(m.nnz, dtype=np.int64) - np.repeat(new_ptr[:-1], counts) + np.repeat(rp[perm], counts)
           if m.nnz else np.zeros(0, dtype=np.int64))
    return CsrMatrix(m.rows, m.cols, new_ptr, to_host(m.col_idx)[src], to_host(m.values)[src])


def spmv_preprocess(m: CsrMatrix, platform: Platform, share: WorkShare | None = None) -> SpmvPrep:
    """Stable sort of rows by nnz, then split_row: the nnz-balanced point of
    the two modeled throughputs, or `searchsorted(cum, f·total, 'left')` for
    an explicit share (:186-203).  Device matrices are permuted on the host
    index arrays and re-uploaded (one-time prep)."""
    if m.on_device:
        perm, permuted = _device_preprocess(m)
        cum = to_host(permuted.row_ptr).astype(np.float64)
    else:
        row_nnz = m.row_nnz
        perm = np.argsort(row_nnz, kind="stable")
        permuted = _permute_rows_host(m, perm)
        cum = np.zeros(m.rows + 1, dtype=np.float64)
        np.cumsum(row_nnz[perm], out=cum[1:])
    total = cum[-1]
    if share is not None:
        split = int(np.searchsorted(cum, share.fraction_a * total, side="left"))
    else:
        t_a = cum / platform.device_a.throughput
        t_b = (total - cum) / platform.device_b.throughput
        split = int(np.argmin(np.maximum(t_a, t_b)))
    return SpmvPrep(permuted, perm, split, platform.device_a.worker_count)


def _device_preprocess(m: CsrMatrix):
    """Row sort + gather on the GPU (hb_spmv_preprocess): returns the
    permutation (int32 CUDA tensor) and the permuted device matrix."""
    import torch

    require_gpu()
    dev = m.row_ptr.device
    perm = torch.empty(m.rows, dtype=torch.int32, device=dev)
    nrp = torch.empty(m.rows + 1, dtype=m.row_ptr.dtype, device=dev)
    ncol = torch.empty_like(m.col_idx)
    nval = torch.empty_like(m.values)
    _lib.call(
        "hb_spmv_preprocess", vp(m.row_ptr.data_ptr()), _index_code(m.row_ptr), vp(m.col_idx.data_ptr()),
        _index_code(m.col_idx), vp(m.values.data_ptr()), m.rows, vp(perm.data_ptr()), _lib.DTYPE_CODES["i4"],
        vp(nrp.data_ptr()), vp(ncol.data_ptr()), vp(nval.data_ptr()), _lib.HB_DEVICE_PTRS, current_stream_handle(nrp),
    )
    return perm, CsrMatrix(m.rows, m.cols, nrp, ncol, nval)


def _host_range_matvec(m: CsrMatrix, x: np.ndarray, row0: int, row1: int, workers: int = 1,
                       perm: Any = None, y: np.ndarray | None = None) -> np.ndarray:
    """DeviceA body (:206-211) in native code (hb_host_spmv_rows on `workers`
    threads): rounded products summed left to right per row — exactly the
    reference's product + bincount arithmetic.  With `perm` and `y`, row r's
    sum goes straight to y[perm[r]] (the un-permute of :224-227 fused in)."""
    if perm is None:
        y = np.zeros(max(row1 - row0, 0))
    if row1 <= row0:
        return y
    rp, ci = buf(to_host(m.row_ptr)), buf(to_host(m.col_idx))
    v = np.ascontiguousarray(to_host(m.values), dtype=np.float64)
    xh = np.ascontiguousarray(x, dtype=np.float64)
    pb = buf(to_host(perm)) if perm is not None else None
    if pb is not None and (pb.code not in (_lib.DTYPE_CODES["i4"], _lib.DTYPE_CODES["i8"]) or y is None
                           or not y.flags.c_contiguous or y.dtype != np.float64):
        raise ValueError("perm must be int32/int64 with a C-contiguous float64 y")
    _lib.call("hb_host_spmv_rows", vp(rp.ptr), rp.code, vp(ci.ptr), ci.code, vp(v.ctypes.data), row0, row1,
              vp(xh.ctypes.data), vp(pb.ptr if pb else 0), pb.code if pb else 0, vp(y.ctypes.data), workers)
    return y
    rp, ci = buf(to_host(m.row_ptr)), buf(to_host(m.col_idx))
    v = np.ascontiguousarray(to_host(m.values), dtype=np.float64)
    xh = np.ascontiguousarray(x, dtype=np.float64)
    _lib.call("hb_host_spmv_rows", vp(rp.ptr), rp.code, vp(ci.ptr), ci.code, vp(v.ctypes.data), row0, row1,
              vp(xh.ctypes.data), vp(y.ctypes.data), workers)
    return y


def gpu_spmv(m: CsrMatrix, x: Any, row0: int, row1: int, y: Any = None, perm: Any = None,
             *, exact: bool = True, method: str | None = None, asynchronous: bool = False) -> Any:
    """DeviceB body (hb_spmv_csr).  Without `perm` returns/fills the y_perm
    slice of rows [row0, row1); with `perm` scatters y[perm[i]] in place.
    `method`: "exact" (default; bit-exact sequential row sums), "warp"
    (warp-per-row tree sums) or "merge" (merge-path, load-balanced for any
    row-length distribution without preprocessing) — the last two within 1e-9
    relative.  `exact=False` is the older spelling of "warp"."""
    _lib.load()
    if row1 > row0:
        require_gpu()
    method = method or ("exact" if exact else "warp")
    modes = {"exact": _lib.HB_SPMV_SEQ, "warp": _lib.HB_SPMV_WARP, "merge": _lib.HB_SPMV_MERGE}
    if method not in modes:
        raise ValueError(f"unknown SpMV method {method!r}")
    mode = modes[method]
    if m.on_device:
        import torch

        if not is_device_array(x):
            x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
        if y is None:
            y = torch.empty(row1 - row0 if perm is None else m.rows, dtype=torch.float64, device=x.device)
        if row1 == row0:
            return y
        flags = _lib.HB_DEVICE_PTRS | (_lib.HB_ASYNC if asynchronous else 0)
        _lib.call(
            "hb_spmv_csr", vp(m.row_ptr.data_ptr()), _index_code(m.row_ptr), vp(m.col_idx.data_ptr()),
            _index_code(m.col_idx), vp(m.values.data_ptr()), row0, row1, m.cols, vp(x.data_ptr()),
            vp(perm.data_ptr() if perm is not None else 0), _index_code(perm) if perm is not None else 0,
            vp(y.data_ptr()), mode, flags, current_stream_handle(x),
        )
        return y
    xb = buf(to_host(x), np.float64)
    rp, ci, v = buf(m.row_ptr), buf(m.col_idx), buf(m.values, np.float64)
    if y is None:
        y = host_empty(row1 - row0 if perm is None else m.rows, np.float64)
    if row1 == row0:
        return y
    pb = buf(perm) if perm is not None else None
    _lib.call(
        "hb_spmv_csr", vp(rp.ptr), _index_code(rp.owner), vp(ci.ptr), _index_code(ci.owner), vp(v.ptr),
        row0, row1, m.cols, vp(xb.ptr), vp(pb.ptr if pb else 0), _index_code(pb.owner) if pb else 0,
        vp(y.ctypes.data), mode, 0, current_stream_handle(),
    )
    return y


def _nnz_bounds(m: CsrMatrix, row0: int, row1: int, world: int) -> list[int]:
    """Device-side partitioner rule for SpMV: G ranges of equal nnz, found by
    the reference's own searchsorted-on-nnz-prefix (:243-245) at k/G."""
    rp = to_host(m.row_ptr).astype(np.float64)
    cum = rp[row0 : row1 + 1] - rp[row0]
    total = cum[-1]
    inner = [row0 + int(np.searchsorted(cum, k * total / world, side="left")) for k in range(1, world)]
    return [row0] + inner + [row1]


def _gpu_rows(m: CsrMatrix, x, row0: int, row1: int) -> np.ndarray:
    g = sharding.active_group()
    if g is None or g.world == 1:
        return sharding.to_numpy(gpu_spmv(m, x, row0, row1))
    b = _nnz_bounds(m, row0, row1, g.world)
    mine = sharding.to_numpy(gpu_spmv(m, x, b[g.rank], b[g.rank + 1]))
    return sharding.allgather_rows(mine, b, g)


def spmv_hybrid(prep: SpmvPrep, x: Any) -> np.ndarray:
    """y = A x with the prep's row split, in original row order (:214-227)."""
    m = prep.permuted
    xh = np.asarray(to_host(x), dtype=np.float64)
    if xh.shape != (m.cols,):
        raise ValueError(f"x must have length {m.cols}, got {xh.shape}")
    split = prep.split_row
    x_side_b = x if (m.on_device and is_device_array(x)) else xh
    g = sharding.active_group()
    if m.on_device or (g is not None and g.world > 1):
        with ThreadPoolExecutor(max_workers=2) as pool:
            fa = pool.submit(_host_range_matvec, m, xh, 0, split, prep.workers_a)
            fb = pool.submit(inherit_device(_gpu_rows), m, x_side_b, split, m.rows)
            y_perm = np.concatenate([fa.result(), fb.result()])
        y = np.empty_like(y_perm)
        y[to_host(prep.perm)] = y_perm
        return y
    # host matrix, one GPU: each side scatters its own rows into y (the GPU
    # side inside the C call) — no concatenation, no full-size host scatter
    perm = np.asarray(to_host(prep.perm))
    y = host_empty(m.rows, np.float64)

    def side_a():
        _host_range_matvec(m, xh, 0, split, prep.workers_a, perm=perm, y=y)

    with ThreadPoolExecutor(max_workers=2) as pool:
        fa = pool.submit(side_a)
        fb = pool.submit(inherit_device(gpu_spmv), m, xh, split, m.rows, y, perm) if split < m.rows else None
        fa.result()
        if fb is not None:
            fb.result()
    return y


class SpmvWorkload:
    """Row-range split of the nnz-sorted matrix, merged back to the original
    row order (:230-257)."""

    name = "spmv"
    unit = "nonzeros"

    def __init__(self, prep: SpmvPrep, x: Any):
        self.prep = prep
        self.x_host = np.asarray(to_host(x), dtype=np.float64)
        if self.x_host.shape != (prep.permuted.cols,):
            raise ValueError("x length must match matrix columns")
        self.x = x if is_device_array(x) else self.x_host
        cum = np.zeros(prep.permuted.rows + 1)
        np.cumsum(prep.permuted.row_nnz, out=cum[1:])
        self._cum = cum

    def partition(self, fraction_a: float):
        split = int(np.searchsorted(self._cum, fraction_a * self._cum[-1], side="left"))
        return (0, split), (split, self.prep.permuted.rows)

    def work_units(self, part) -> float:
        return float(self._cum[part[1]] - self._cum[part[0]])

    def run_part(self, device: Device, part) -> np.ndarray:
        if device.id is DeviceId.B:
            return _gpu_rows(self.prep.permuted, self.x, part[0], part[1])
        return _host_range_matvec(self.prep.permuted, self.x_host, part[0], part[1], device.worker_count)

    def merge(self, partials: Sequence[np.ndarray]) -> np.ndarray:
        y_perm = np.concatenate(partials)
        y = np.empty_like(y_perm)
        y[to_host(self.prep.perm)] = y_perm
        return y


# --------------------------------------------------------------------------
# list ranking (kernels_irregular.py:356-508)


@dataclass(frozen=True)
class LinkedListArr:
    """Successor-array list: succ[i] is the next node or LIST_END (:360-365)."""

    succ: Any
    head: int


@dataclass(frozen=True)
class ListRankStats:
    fis_rounds: int
    round_sizes: tuple[int, ...]
    reduced_size: int
    removed_total: int
    sublist_count: int


def validate_list(lst: LinkedListArr) -> None:
    """The chain from head must visit every node exactly once (:377-393).
    Host arrays: range check + walk on the host like the reference; CUDA
    tensors: the GPU ranking itself validates (hb_list_rank)."""
    succ = lst.succ
    n = int(succ.numel() if is_device_array(succ) else succ.size)
    if not 0 <= lst.head < n:
        raise StructuralError("head out of range")
    if is_device_array(succ):
        gpu_list_rank(succ, lst.head)
        return
    if n and (succ.min() < LIST_END or succ.max() >= n):
        raise StructuralError("successor index out of range")
    seen, cur = 0, lst.head
    while cur != LIST_END:
        seen += 1
        if seen > n:
            raise StructuralError("list contains a cycle")
        cur = int(succ[cur])
    if seen != n:
        raise StructuralError(f"chain covers {seen} of {n} nodes (broken list)")


def gpu_list_rank(succ: Any, head: int, out: Any = None, *, asynchronous: bool = False) -> Any:
    """rank[i] = distance of node i from `head` (hb_list_rank: sparse ruling
    set + Wyllie pointer jumping).  Host succ → int64 numpy ranks; CUDA succ
    (int32/int64) → int64 CUDA tensor.  Malformed lists raise StructuralError."""
    _lib.load()
    require_gpu()
    sb = buf(succ)
    if sb.dtype not in (np.dtype(np.int32), np.dtype(np.int64)):
        sb = buf(np.asarray(to_host(succ), dtype=np.int64))
    n = sb.size
    if n < 1:
        raise StructuralError("head out of range")
    code = _index_code(sb.owner)
    if sb.device:
        import torch

        res = out if out is not None else torch.empty(n, dtype=torch.int64, device=succ.device)
        flags = _lib.HB_DEVICE_PTRS | (_lib.HB_ASYNC if asynchronous else 0)
        _lib.call("hb_list_rank", vp(sb.ptr), code, n, int(head), vp(res.data_ptr()), flags,
                  current_stream_handle(succ))
        return res
    res = host_empty(n, np.int64)
    _lib.call("hb_list_rank", vp(sb.ptr), code, n, int(head), vp(res.ctypes.data), 0, current_stream_handle())
    return res


def gpu_list_fis_stats(succ: Any, head: int, seed: int, sublists: int) -> ListRankStats:
    """The reference's FIS reduction + sublist-head choice on the GPU
    (hb_list_fis_stats), for its ListRankStats (:396-448, :495-501)."""
    _lib.load()
    require_gpu()
    sb = buf(succ)
    if sb.dtype not in (np.dtype(np.int32), np.dtype(np.int64)):
        sb = buf(np.asarray(to_host(succ), dtype=np.int64))
    cap = 1000
    sizes = np.zeros(cap, dtype=np.int64)
    st = np.zeros(4, dtype=np.int64)
    flags = _lib.HB_DEVICE_PTRS if sb.device else 0
    _lib.call("hb_list_fis_stats", vp(sb.ptr), _index_code(sb.owner), sb.size, int(head), int(seed) & ((1 << 64) - 1),
              int(sublists), vp(sizes.ctypes.data), cap, vp(st.ctypes.data), flags,
              current_stream_handle(succ if sb.device else None))
    rounds = int(st[0])
    return ListRankStats(rounds, tuple(int(v) for v in sizes[:rounds]), int(st[1]), int(st[2]), int(st[3]))


def list_rank_with_stats(lst: LinkedListArr, platform: Platform, seed: int) -> tuple[Any, ListRankStats]:
    """(rank, ListRankStats) like the reference (:481-502).  Ranks: GPU sparse
    ruling set (validates the list first, StructuralError as validate_list);
    statistics: the reference's own FIS reduction and sublist choice, on the
    GPU, with sublists = 4 x (workers_a + workers_b)."""
    rank = gpu_list_rank(lst.succ, lst.head)
    workers = platform.device_a.worker_count + platform.device_b.worker_count
    stats = gpu_list_fis_stats(lst.succ, lst.head, seed, 4 * workers)
    return rank, stats


def list_rank_hybrid(lst: LinkedListArr, platform: Platform, seed: int) -> Any:
    """rank[i] = distance of node i from the head (:505-508).  The ranks do
    not depend on the seed or on the reduction schedule, so this entry point
    takes the GPU fast path directly (validation included)."""
    return gpu_list_rank(lst.succ, lst.head)
