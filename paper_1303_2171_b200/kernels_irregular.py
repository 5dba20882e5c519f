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


def sell_layout(m: CsrMatrix):
    """The SELL-32 copy of a device int32 matrix (hb_spmv_sell_build), built
    once and cached on the matrix (device matrices are not mutated in place):
    (tile_off int64[ntiles+1], col int32[total], val float64[total])."""
    import ctypes

    import torch

    cached = getattr(m, "_sell", None)
    if cached is not None:
        return cached
    ntiles = (m.rows + 31) // 32
    dev = m.row_ptr.device
    toff = torch.empty(ntiles + 1, dtype=torch.int64, device=dev)
    total = ctypes.c_int64(0)
    st = current_stream_handle(m.row_ptr)
    _lib.call("hb_spmv_sell_build", vp(m.row_ptr.data_ptr()), None, None, m.rows, vp(toff.data_ptr()), None, None,
              ctypes.byref(total), _lib.HB_DEVICE_PTRS, st)
    scol = torch.empty(total.value, dtype=torch.int32, device=dev)
    sval = torch.empty(total.value, dtype=torch.float64, device=dev)
    _lib.call("hb_spmv_sell_build", vp(m.row_ptr.data_ptr()), vp(m.col_idx.data_ptr()), vp(m.values.data_ptr()),
              m.rows, vp(toff.data_ptr()), vp(scol.data_ptr()), vp(sval.data_ptr()), ctypes.byref(total),
              _lib.HB_DEVICE_PTRS, st)
    layout = (toff, scol, sval)
    object.__setattr__(m, "_sell", layout)
    return layout


def gpu_spmv(m: CsrMatrix, x: Any, row0: int, row1: int, y: Any = None, perm: Any = None,
             *, exact: bool = True, method: str | None = None, asynchronous: bool = False) -> Any:
    """DeviceB body (hb_spmv_csr).  Without `perm` returns/fills the y_perm
    slice of rows [row0, row1); with `perm` scatters y[perm[i]] in place.
    `method`: "exact" (default; bit-exact sequential row sums — on a device
    int32 matrix through its cached SELL-32 copy, `sell_layout`),
    "exact_csr" (the same arithmetic straight from the CSR arrays), "warp"
    (warp-per-row tree sums) or "merge" (merge-path, load-balanced for any
    row-length distribution without preprocessing) — the last two within 1e-9
    relative.  `exact=False` is the older spelling of "warp"."""
    _lib.load()
    if row1 > row0:
        require_gpu()
    method = method or ("exact" if exact else "warp")
    modes = {"exact": _lib.HB_SPMV_SEQ, "exact_csr": _lib.HB_SPMV_SEQ, "warp": _lib.HB_SPMV_WARP,
             "merge": _lib.HB_SPMV_MERGE}
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
        if method == "exact" and m.row_ptr.dtype == torch.int32 and m.col_idx.dtype == torch.int32:
            toff, scol, sval = sell_layout(m)
            _lib.call("hb_spmv_sell", vp(m.row_ptr.data_ptr()), vp(toff.data_ptr()), vp(scol.data_ptr()),
                      vp(sval.data_ptr()), row0, row1, vp(x.data_ptr()),
                      vp(perm.data_ptr() if perm is not None else 0), _index_code(perm) if perm is not None else 0,
                      vp(y.data_ptr()), flags, current_stream_handle(x))
            return y
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


def nnz_bounds_host(row_ptr: np.ndarray, row0: int, row1: int, parts: int) -> list[int]:
    """SpmvWorkload's split rule (:243-245) at k/G on a host row_ptr:
    G row ranges of equal nnz, searchsorted(cum, k·total/G, 'left')."""
    cum = np.asarray(row_ptr[row0 : row1 + 1], dtype=np.float64) - float(row_ptr[row0])
    total = cum[-1]
    inner = [row0 + int(np.searchsorted(cum, k * total / parts, side="left")) for k in range(1, parts)]
    return [row0] + inner + [row1]


def partition_nnz(m: CsrMatrix, row0: int, row1: int, parts: int) -> list[int]:
    """The device-side partitioner: G+1 row bounds of equal nnz over rows
    [row0, row1).  Device matrices: hb_partition_nnz binary-searches the
    device row_ptr (only the G+1 bounds come back); host matrices: the same
    rule on the host array (nothing to copy)."""
    if parts == 1:
        return [row0, row1]
    if not m.on_device:
        return nnz_bounds_host(m.row_ptr, row0, row1, parts)
    out = np.zeros(parts + 1, dtype=np.int64)
    _lib.call("hb_partition_nnz", vp(m.row_ptr.data_ptr()), _index_code(m.row_ptr), row0, row1, parts,
              vp(out.ctypes.data), _lib.HB_DEVICE_PTRS, current_stream_handle(m.row_ptr))
    return [int(v) for v in out]


def scatter_perm(src: Any, perm: Any, dst: Any) -> Any:
    """dst[perm[i]] = src[i] on the device (hb_scatter_perm; the un-permute
    of SpmvWorkload.merge, :253-257)."""
    n = int(src.numel())
    if n:
        _lib.call("hb_scatter_perm", vp(src.data_ptr()), n, src.element_size(), vp(perm.data_ptr()),
                  _index_code(perm), vp(dst.data_ptr()), _lib.HB_DEVICE_PTRS, current_stream_handle(src))
    return dst


def _gpu_rows(m: CsrMatrix, x, row0: int, row1: int) -> Any:
    """DeviceB rows [row0, row1) → y_perm slice (numpy for a host matrix,
    CUDA tensor for a device matrix).  Under a GPU group: equal-nnz shards
    from the device-side partitioner, one all-gather of the y slices."""
    g = sharding.active_group()
    if not sharding.multi(g):
        return gpu_spmv(m, x, row0, row1)
    b = partition_nnz(m, row0, row1, g.world)
    mine = gpu_spmv(m, x, b[g.rank], b[g.rank + 1])
    return sharding.gather_rows(mine, b, g)


def _spmv_device(prep: SpmvPrep, x: Any) -> Any:
    """spmv_hybrid for a device-resident matrix: y stays in HBM.  One GPU:
    the kernel stores y[perm[i]] directly (fused un-permute).  GPU group:
    every rank computes its equal-nnz shard of y_perm, all-gather, then
    hb_scatter_perm.  A host share (split_row > 0) runs on the host cores
    and is scattered in on the device."""
    import torch

    m = prep.permuted
    xd = x if is_device_array(x) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(m.row_ptr.device)
    perm = prep.perm
    if not is_device_array(perm):
        perm = torch.from_numpy(np.ascontiguousarray(perm, dtype=np.int64)).to(xd.device)
    split = prep.split_row
    y = torch.empty(m.rows, dtype=torch.float64, device=xd.device)
    g = sharding.active_group()
    pool = ThreadPoolExecutor(max_workers=1) if split else None  # the host share runs beside the GPU rows
    try:
        fa = pool.submit(_host_range_matvec, m.to_host(), np.asarray(to_host(xd)), 0, split, prep.workers_a) if pool else None
        if split < m.rows:
            if sharding.multi(g):
                scatter_perm(_gpu_rows(m, xd, split, m.rows), perm[split:], y)
            else:
                gpu_spmv(m, xd, split, m.rows, y=y, perm=perm)
        if fa is not None:
            scatter_perm(torch.from_numpy(fa.result()).to(y.device), perm[:split], y)
    finally:
        if pool is not None:
            pool.shutdown()
    return y if is_device_array(x) else y.cpu().numpy()


def spmv_hybrid(prep: SpmvPrep, x: Any) -> Any:
    """y = A x with the prep's row split, in original row order (:214-227).
    Host matrix → numpy y; device matrix → y computed in HBM (a CUDA tensor
    when x is one, else copied back to numpy)."""
    m = prep.permuted
    if not is_device_array(x):
        x = np.asarray(x, dtype=np.float64)
    if tuple(x.shape) != (m.cols,):
        raise ValueError(f"x must have length {m.cols}, got {tuple(x.shape)}")
    if m.on_device:
        return _spmv_device(prep, x)
    xh = np.asarray(to_host(x), dtype=np.float64)
    split = prep.split_row
    g = sharding.active_group()
    if sharding.multi(g):
        with ThreadPoolExecutor(max_workers=2) as pool:
            fa = pool.submit(_host_range_matvec, m, xh, 0, split, prep.workers_a)
            fb = pool.submit(inherit_device(_gpu_rows), m, xh, split, m.rows)
            y_perm = np.concatenate([fa.result(), sharding.to_numpy(fb.result())])
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

    def merge(self, partials: Sequence[Any]) -> np.ndarray:
        y_perm = np.concatenate([sharding.to_numpy(p) for p in partials])
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
    if sharding.multi():
        return list_rank_sharded(succ, head, sharding.active_group(), out)
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


def list_rank_sharded(succ: Any, head: int, g: "sharding.ShardGroup", out: Any = None) -> Any:
    """List ranking over a GPU group — the sublist split of the reference's
    _rank_reduced (:431-478) mapped onto GPUs: succ replicated
    on every rank; the level-1 sublists (every 64th node + the head) split
    floor(k·S/G) by id; each rank walks its own (hb_lr_walk_part); the
    (next, length) summaries are all-gathered; every rank ranks the sublist
    chain and expands the ranks of its own nodes (hb_lr_finish_part, 0 for
    the others); an all-reduce (sum) leaves every rank with all ranks.
    Errors (bad successors, cycles, broken lists) are detected identically
    on every rank, so no rank is left waiting in a collective."""
    import ctypes

    import torch

    n = int(succ.numel() if is_device_array(succ) else np.asarray(succ).size)
    if not 0 <= head < max(n, 1) or n < 1:
        raise StructuralError("head out of range")
    if is_device_array(succ):
        sd = succ if succ.dtype in (torch.int32, torch.int64) else succ.to(torch.int64)
    else:
        host = np.asarray(succ)
        if host.size and (host.min() < LIST_END or host.max() >= n):
            raise StructuralError("successor index out of range")
        sd = torch.from_numpy(np.ascontiguousarray(host, dtype=np.int32 if n < 2**31 else np.int64)).cuda()
    sd = sd.contiguous()
    nsub, sub_head = ctypes.c_int64(0), ctypes.c_int64(0)
    _lib.call("hb_lr_layout", n, int(head), ctypes.byref(nsub), ctypes.byref(sub_head))
    nsub, sub_head = nsub.value, sub_head.value
    b = sharding.shard_bounds(nsub, g.world)
    lo, hi = b[g.rank], b[g.rank + 1]
    dev = sd.device
    rank = out if out is not None else torch.empty(n, dtype=torch.int64, device=dev)
    nxt = torch.empty(nsub, dtype=torch.int64, device=dev)
    ln = torch.empty(nsub, dtype=torch.int64, device=dev)
    stream = current_stream_handle(sd)
    _lib.call("hb_lr_walk_part", vp(sd.data_ptr()), _index_code(sd), n, int(head), lo, hi, vp(rank.data_ptr()),
              vp(nxt.data_ptr()), vp(ln.data_ptr()), _lib.HB_DEVICE_PTRS | _lib.HB_ASYNC, stream)
    counts = [b[k + 1] - b[k] for k in range(g.world)]
    nxt_all = sharding.gather_blocks(nxt[lo:hi], counts, g)
    ln_all = sharding.gather_blocks(ln[lo:hi], counts, g)
    flags = _lib.HB_DEVICE_PTRS | _lib.HB_ASYNC
    if n <= 2**31:  # int32 ranks on the wire: the merging all-reduce moves 4 bytes per node, not 8
        r32 = torch.empty(n, dtype=torch.int32, device=dev)
        _lib.call("hb_lr_finish_part32", vp(nxt_all.data_ptr()), vp(ln_all.data_ptr()), nsub, sub_head, n, lo, hi,
                  vp(rank.data_ptr()), vp(r32.data_ptr()), flags, stream)
        sharding.all_reduce_sum(r32, g)
        _lib.call("hb_widen_i32", vp(r32.data_ptr()), n, vp(rank.data_ptr()), flags, current_stream_handle(r32))
    else:
        _lib.call("hb_lr_finish_part", vp(nxt_all.data_ptr()), vp(ln_all.data_ptr()), nsub, sub_head, n, lo, hi,
                  vp(rank.data_ptr()), flags, stream)
        sharding.all_reduce_sum(rank, g)
    return rank if is_device_array(succ) else rank.cpu().numpy()


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
