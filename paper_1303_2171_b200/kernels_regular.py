"""Regular hot-path kernels behind the reference's own entry points
(hybridbench/kernels_regular.py): histogram, sort, convolution, bilateral
filter.

Each workload keeps the reference's Partitionable protocol and names.
`run_part(DeviceA, …)` computes the host share with numpy on the host
cores; `run_part(DeviceB, …)` is the GPU share, one libhb200 call (sharded
over the active GPU group, see sharding.py).  Inputs may be numpy arrays
(host; staged inside the C call) or CUDA tensors (device-resident).
"""

from __future__ import annotations

import math
import re
from dataclasses import dataclass
from pathlib import Path
from typing import Any, Sequence

import numpy as np

from . import _lib, sharding
from .errors import DataIOError
from .gpu import (buf, current_stream_handle, flags_for, host_empty, inherit_device, is_device_array, require_gpu,
                  result_scope, to_host, vp)
from .platform import Device, DeviceId, Platform
from .worksharing import WorkShare, formula_share, run_workshared

# --------------------------------------------------------------------------
# images


@dataclass(frozen=True)
class Image:
    """Row-major pixel grid: uint8 inputs, float outputs (kernels_regular.py:29-45)."""

    pixels: Any

    def __post_init__(self) -> None:
        shape = tuple(self.pixels.shape)
        if len(shape) != 2 or shape[0] * shape[1] == 0:
            raise ValueError("pixels must be a non-empty 2-D array")

    @property
    def height(self) -> int:
        return int(self.pixels.shape[0])

    @property
    def width(self) -> int:
        return int(self.pixels.shape[1])


def read_pgm(path: str | Path) -> Image:
    """kernels_regular.py:48-69: P5 (binary) or P2 (ASCII) PGM, maxval <= 255,
    '#' comments in the header; any failure → DataIOError."""
    try:
        raw = Path(path).read_bytes()
    except OSError as exc:
        raise DataIOError(f"cannot read image {path}: {exc}") from exc
    try:
        magic, (width, height, maxval), start = _parse_pgm_header(raw)
        if not 0 < maxval <= 255:
            raise ValueError(f"unsupported maxval {maxval}")
        count = width * height
        if magic == b"P5":
            pix = np.frombuffer(raw, dtype=np.uint8, count=count, offset=start)
        else:
            tokens = raw[start:].split()
            if len(tokens) < count:
                raise ValueError("truncated P2 payload")
            pix = np.array([int(t) for t in tokens[:count]], dtype=np.uint8)
        return Image(pix.reshape(height, width).copy())
    except Exception as exc:
        raise DataIOError(f"malformed PGM {path}: {exc}") from exc


def _parse_pgm_header(raw: bytes) -> tuple[bytes, tuple[int, int, int], int]:
    """Magic, (width, height, maxval) and the payload offset: three integer
    fields separated by whitespace and '#'-to-end-of-line comments, then
    exactly one whitespace byte before the payload (:72-91)."""
    magic = raw[:2]
    if magic not in (b"P2", b"P5"):
        raise ValueError("not a P2/P5 PGM")
    fields: list[int] = []
    pos = 2
    while len(fields) < 3:
        m = re.compile(rb"(?:\s|#[^\n]*)*").match(raw, pos)
        pos = m.end()
        tok = re.compile(rb"\S+").match(raw, pos)
        if tok is None:
            raise ValueError("truncated PGM header")
        fields.append(int(tok.group()))
        pos = tok.end()
    return magic, (fields[0], fields[1], fields[2]), pos + 1


def write_pgm(image: Image, path: str | Path, binary: bool = True) -> None:
    """kernels_regular.py:94-110: maxval-255 PGM; non-uint8 pixels are rounded
    half-to-even and clamped to [0, 255]."""
    data = sharding.to_numpy(image.pixels)
    if data.dtype != np.uint8:
        data = np.clip(np.rint(data), 0, 255).astype(np.uint8)
    head = ("P5" if binary else "P2") + f"\n{image.width} {image.height}\n255\n"
    try:
        with open(path, "wb") as fh:
            fh.write(head.encode("ascii"))
            if binary:
                fh.write(np.ascontiguousarray(data).tobytes())
            else:
                fh.write("".join(" ".join(map(str, row.tolist())) + "\n" for row in data).encode("ascii"))
    except OSError as exc:
        raise DataIOError(f"cannot write image {path}: {exc}") from exc


# --------------------------------------------------------------------------
# histogram (kernels_regular.py:116-169)


@dataclass(frozen=True)
class HistogramResult:
    bins: np.ndarray
    bin_count: int

    def __post_init__(self) -> None:
        if self.bin_count < 1 or len(self.bins) != self.bin_count:
            raise ValueError("bins length must equal bin_count >= 1")


def _dtype_within(dtype: np.dtype, bin_count: int) -> bool:
    """True when every value of `dtype` is a valid bin (no check needed)."""
    if dtype.kind == "u" and dtype.itemsize <= 4:
        return (1 << (8 * dtype.itemsize)) <= bin_count
    if dtype.kind == "b":
        return bin_count >= 2
    return False


def gpu_histogram(part: Any, bin_count: int, out: Any = None, *, asynchronous: bool = False) -> Any:
    """Bin counts of `part` on the GPU (hb_hist; replaces the DeviceB body of
    HistogramWorkload.run_part, kernels_regular.py:149-154).

    Host input → int64 numpy counts.  CUDA-tensor input → counts written to
    `out` (int64 CUDA tensor, allocated when None) and returned; with
    `asynchronous=True` nothing is synchronised (for graph capture/timing)."""
    b = buf(part)
    if b.size or b.device:
        require_gpu()
    _lib.load()
    if b.code == 0 or b.dtype.kind == "f":
        raise TypeError(f"histogram input must be an integer array, got {b.dtype}")
    if b.device:
        import torch

        res = out if out is not None else torch.empty(bin_count, dtype=torch.int64, device=part.device)
        _lib.call(
            "hb_hist", vp(b.ptr), b.code, b.size, bin_count, vp(res.data_ptr()),
            flags_for(b, asynchronous=asynchronous), current_stream_handle(part),
        )
        return res
    res = np.zeros(bin_count, dtype=np.int64)
    _lib.call("hb_hist", vp(b.ptr), b.code, b.size, bin_count, vp(res.ctypes.data), 0, current_stream_handle())
    return res


def host_histogram(part: Any, bin_count: int, workers: int = 1) -> np.ndarray:
    """DeviceA body (kernels_regular.py:149-154): per-worker private counts on
    `workers` host threads (hb_host_hist, native), summed; int64 counts."""
    b = buf(to_host(part))
    if b.code == 0 or b.dtype.kind == "f":
        raise TypeError(f"histogram input must be an integer array, got {b.dtype}")
    res = np.zeros(bin_count, dtype=np.int64)
    _lib.call("hb_host_hist", vp(b.ptr), b.code, b.size, bin_count, vp(res.ctypes.data), workers)
    return res


class HistogramWorkload:
    """Index-range split (kernels_regular.py:126-160).  DeviceA: per-worker
    private numpy histograms; DeviceB: the privatised smem GPU kernel, its
    share further split over the GPU group and summed with a collective."""

    name = "hist"
    unit = "elements"

    def __init__(self, data: Any, bin_count: int):
        if bin_count < 1:
            raise ValueError("bin_count must be >= 1")
        if not is_device_array(data):
            data = np.asarray(data)
        size = int(data.numel() if is_device_array(data) else data.size)
        if size and not is_device_array(data) and not _dtype_within(data.dtype, bin_count):
            if data.min() < 0 or data.max() >= bin_count:
                raise ValueError("element outside bin domain")
        # device tensors: the GPU kernel checks the domain in-line and raises
        # the same ValueError from run_part (no extra pass over HBM)
        self.data = data
        self.bin_count = bin_count

    def partition(self, fraction_a: float):
        n = int(self.data.numel() if is_device_array(self.data) else self.data.size)
        split = int(math.floor(fraction_a * n))
        return self.data[:split], self.data[split:]

    def work_units(self, part) -> float:
        return float(part.numel() if is_device_array(part) else part.size)

    def run_part(self, device: Device, part) -> np.ndarray:
        if device.id is DeviceId.B:
            return sharding.run_sharded_histogram(part, self.bin_count)
        return host_histogram(part, self.bin_count, device.worker_count)

    def merge(self, partials: Sequence[Any]) -> HistogramResult:
        total = np.zeros(self.bin_count, dtype=np.int64)
        for p in partials:
            total += sharding.to_numpy(p)
        return HistogramResult(total, self.bin_count)


def hybrid_histogram(
    data: Any, bin_count: int, platform: Platform, share: WorkShare | None = None
) -> HistogramResult:
    """kernels_regular.py:163-169: work-shared histogram, no baselines."""
    workload = HistogramWorkload(data, bin_count)
    result, _ = run_workshared(platform, workload, share or formula_share(platform), baselines=False)
    return result


# --------------------------------------------------------------------------
# sort (kernels_regular.py:172-321)

SORT_FANOUT = 64
SORT_HIST_CELLS = 256
SORT_MAX_DEPTH = 8

_SORT_CODES = {np.dtype(np.uint32): 5, np.dtype(np.int32): 6, np.dtype(np.uint64): 7, np.dtype(np.int64): 8}


def gpu_sort(keys: Any, payload: Any = None, *, asynchronous: bool = False,
             ballot: bool = False) -> tuple[Any, Any, int]:
    """LSD radix sort on the GPU (hb_sort).  CUDA tensors are sorted in place
    (payload permuted alongside, stably); host arrays are left untouched and
    sorted copies returned.  Returns (keys, payload, digit passes executed;
    None for asynchronous device sorts, which do not wait to learn it).
    `ballot` ranks with the ballot multi-split instead of the (device-checked)
    lane-ordered shared atomics."""
    import ctypes

    _lib.load()
    kb = buf(keys)
    code = _SORT_CODES.get(kb.dtype)
    if code is None:
        raise TypeError(f"sort keys must be u32/i32/u64/i64, got {kb.dtype}")
    if kb.size > 1 or kb.device:
        require_gpu()
    vb = None
    if payload is not None:
        vb = buf(payload) if is_device_array(payload) else buf(payload, np.uint32)
        if vb.dtype not in (np.dtype(np.uint32), np.dtype(np.int32)) or vb.size != kb.size:
            raise TypeError("payload must be uint32 (or non-negative int32) with one entry per key")
    flags = flags_for(kb, *([vb] if vb else []), asynchronous=asynchronous) | (_lib.HB_SORT_BALLOT if ballot else 0)
    if kb.device:
        k_out, v_out = kb.ptr, (vb.ptr if vb else 0)
        res_k, res_v = keys, payload
    else:
        with result_scope():
            res_k = host_empty(kb.owner.shape, kb.dtype)
            res_v = host_empty(kb.size, vb.dtype) if vb else None
        k_out, v_out = res_k.ctypes.data, (res_v.ctypes.data if vb else 0)
    # asynchronous device sorts do not ask for the pass count: reading it
    # would wait on the digit histogram mid-call (32-bit keys then never
    # block the host and are CUDA-graph capturable); passes is None then
    want_passes = not (asynchronous and kb.device)
    passes = ctypes.c_int32(0)
    _lib.call("hb_sort", vp(kb.ptr), vp(k_out), code, vp(vb.ptr if vb else 0), vp(v_out), kb.size,
              ctypes.byref(passes) if want_passes else None, flags,
              current_stream_handle(keys if kb.device else None))
    return res_k, res_v, (passes.value if want_passes else None)


def _cell_indices(chunk: np.ndarray, lo, hi) -> np.ndarray:
    scale = SORT_HIST_CELLS / (float(hi) - float(lo))
    return np.clip(((chunk - float(lo)) * scale).astype(np.int64), 0, SORT_HIST_CELLS - 1)


def _quantile_splitters(counts: np.ndarray, n: int, lo, hi) -> np.ndarray:
    cum = np.cumsum(counts)
    cells = np.searchsorted(cum, np.arange(1, SORT_FANOUT) * (n / SORT_FANOUT), side="left")
    return np.unique(float(lo) + (cells + 1) * ((float(hi) - float(lo)) / SORT_HIST_CELLS))


def _host_sort_plan(arr: np.ndarray, fraction: float):
    """The reference's hybrid binning and smallest-bins-first cut
    (kernels_regular.py:264-292): returns (bin_ids, bin_sizes, on_a)."""
    n = arr.size
    lo, hi = arr.min(), arr.max()
    split = int(math.floor(fraction * n))
    cells = _cell_indices(arr, lo, hi)
    counts = np.bincount(cells[:split], minlength=SORT_HIST_CELLS) + np.bincount(cells[split:], minlength=SORT_HIST_CELLS)
    spl = _quantile_splitters(counts, n, lo, hi)
    ids = np.searchsorted(spl, arr, side="right")
    sizes = np.bincount(ids, minlength=spl.size + 1)
    asc = np.argsort(sizes, kind="stable")
    prefix = np.concatenate([[0.0], np.cumsum(sizes[asc])])
    cut = int(np.argmin(np.maximum(prefix / fraction, (n - prefix) / (1.0 - fraction))))
    on_a = np.zeros(sizes.size, dtype=bool)
    on_a[asc[:cut]] = True
    return ids, sizes, on_a


_F_TOP = {8: np.uint64(1 << 63), 4: np.uint32(1 << 31)}


def _sortable(arr: np.ndarray):
    """(keys the GPU radix sort takes, function mapping sorted keys back).
    u32/i32/u64/i64 go as they are; narrower integers and bools are widened
    (and cast back); floats become order-preserving unsigned bit patterns
    (sign bit set → all bits flipped, else the sign bit set), which sort
    exactly like the values (-0.0 before +0.0) and map back bit for bit."""
    dt = arr.dtype
    if dt in _SORT_CODES:
        return arr, lambda k: k
    if dt.kind == "b" or (dt.kind in "ui" and dt.itemsize < 4):
        wide = np.int32 if dt.kind == "i" else np.uint32
        return arr.astype(wide), lambda k: np.asarray(k).astype(dt)
    if dt.kind == "f":
        src = arr.astype(np.float32) if dt.itemsize < 4 else arr
        width = src.dtype.itemsize
        ut = np.uint64 if width == 8 else np.uint32
        top = _F_TOP[width]
        bits = src.view(ut)
        neg = (bits >> ut(8 * width - 1)).astype(bool)
        keys = np.where(neg, ~bits, bits | top)

        def back(k):
            k = np.asarray(k)
            orig = np.where((k & top).astype(bool), k ^ top, ~k).astype(ut)
            return orig.view(src.dtype).astype(dt)

        return keys, back
    raise TypeError(f"cannot sort keys of dtype {dt}")


def _sortable_tensor(t: Any):
    """The same for CUDA tensors (torch ops on the device)."""
    import torch

    if t.dtype in (torch.int32, torch.int64) or t.dtype in (getattr(torch, "uint32", None), getattr(torch, "uint64", None)):
        return t, lambda k: k
    if t.dtype in (torch.uint8, torch.bool):
        return t.to(torch.int32), lambda k: k.to(t.dtype)
    if t.dtype in (torch.int8, torch.int16):
        return t.to(torch.int32), lambda k: k.to(t.dtype)
    if t.dtype in (torch.float16, torch.bfloat16, torch.float32, torch.float64):
        src = t if t.dtype in (torch.float32, torch.float64) else t.to(torch.float32)
        st = torch.int64 if src.dtype == torch.float64 else torch.int32
        low = torch.iinfo(st).max  # every bit but the sign
        shift = 8 * src.element_size() - 1
        # negative floats: flip all but the sign bit → the signed integer order
        # is the float order; the map is its own inverse
        keys = src.view(st) ^ ((src.view(st) >> shift) & low)

        def back(k):
            return (k ^ ((k >> shift) & low)).view(src.dtype).to(t.dtype)

        return keys, back
    raise TypeError(f"cannot sort keys of dtype {t.dtype}")


def sample_sort_hybrid(
    data: Any, platform: Platform, leaf_a: int = 2048, leaf_b: int = 32, share: WorkShare | None = None
) -> tuple[Any, float, float]:
    """kernels_regular.py:239-310 → (sorted, work_a, work_b), same work
    accounting.  DeviceA sorts its bins with numpy on the host; DeviceB's bins
    are radix-sorted on the GPU (one LSD sort of their union — the bins are
    disjoint value ranges, so that equals sorting each bin), sharded over the
    GPU group with a sample-merge exchange when one is active."""
    if not leaf_a >= leaf_b >= 2:
        raise ValueError("need leaf_a >= leaf_b >= 2")
    fraction = (share or formula_share(platform)).fraction_a
    dev = is_device_array(data)
    arr = data if dev else np.asarray(data)
    n = int(arr.numel() if dev else arr.size)
    if n <= 1:
        return (arr.clone() if dev else arr.copy()), float(n), 0.0
    if n <= leaf_a:
        host = np.sort(to_host(arr), kind="quicksort")
        return _like(host, data), float(n), 0.0
    if fraction <= 0.0:
        # every bin on DeviceB: one GPU sort; a constant array is the
        # reference's lo == hi early return (work on DeviceA)
        keys, back = _sortable_tensor(arr) if dev else _sortable(arr)
        out, _, passes = sharding.run_sharded_sort(keys.clone() if dev and keys is arr else keys)
        out = back(out)
        if passes == 0:
            return out, float(n), 0.0
        return out, 0.0, float(n)
    host = to_host(arr)
    lo, hi = host.min(), host.max()
    if lo == hi:
        return (arr.clone() if dev else arr.copy()), float(n), 0.0
    if fraction >= 1.0:
        return _like(np.sort(host, kind="quicksort"), data), float(n), 0.0
    ids, sizes, on_a = _host_sort_plan(host, fraction)
    mask_a = on_a[ids]
    part_a, part_b = host[mask_a], host[~mask_a]
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=2) as pool:
        fa = pool.submit(np.sort, part_a, kind="quicksort")
        keys_b, back_b = _sortable(part_b)
        fb = pool.submit(inherit_device(lambda: back_b(sharding.to_numpy(sharding.run_sharded_sort(keys_b)[0]))))
        sorted_a, sorted_b = fa.result(), fb.result()
    out = np.empty_like(host)
    pos = pa = pb = 0
    for i, size in enumerate(sizes.tolist()):
        if on_a[i]:
            out[pos : pos + size] = sorted_a[pa : pa + size]
            pa += size
        else:
            out[pos : pos + size] = sorted_b[pb : pb + size]
            pb += size
        pos += size
    work_a = float(sizes[on_a].sum())
    return _like(out, data), work_a, float(n) - work_a


def _like(host: np.ndarray, ref: Any) -> Any:
    if is_device_array(ref):
        import torch

        return torch.from_numpy(np.ascontiguousarray(host)).to(ref.device)
    return host


def hybrid_sort(data: Any, platform: Platform, leaf_a: int = 2048, leaf_b: int = 32,
                share: WorkShare | None = None) -> Any:
    """kernels_regular.py:313-321."""
    out, _, _ = sample_sort_hybrid(data, platform, leaf_a, leaf_b, share)
    return out


# --------------------------------------------------------------------------
# row-strip filters: shared output image


def _host_rows_out(out: np.ndarray | None, rows: int, width: int) -> np.ndarray:
    if out is None:
        return np.zeros((max(rows, 0), width))
    if out.shape != (max(rows, 0), width) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 (rows, width) array")
    return out


class _StripOutput:
    """Both sides of a host-image run write their row strips straight into one
    output image allocated by partition() (host_empty: pinned, so the GPU
    strip lands by DMA), so merge() hands that image back instead of the
    reference's vstack copy (an extra pass over H×W×8 bytes).  Device images
    and GPU groups keep the partial-array protocol."""

    def _new_output(self, height: int, width: int) -> None:
        pix = self.image.pixels
        local = not is_device_array(pix) and (sharding.active_group() is None or sharding.active_group().world == 1)
        self._out = host_empty((height, width)) if local else None

    def _strip(self, part) -> np.ndarray | None:
        out = getattr(self, "_out", None)
        return None if out is None else out[part[0] : part[1]]

    def merge(self, partials: Sequence[np.ndarray]) -> Image:
        out = getattr(self, "_out", None)
        if out is not None and all(isinstance(p, np.ndarray) and (p.size == 0 or np.shares_memory(p, out))
                                   for p in partials):
            return Image(out)
        return Image(np.vstack([sharding.to_numpy(p) for p in partials]))


# --------------------------------------------------------------------------
# convolution (kernels_regular.py:327-414)


@dataclass(frozen=True)
class FilterKernel:
    """Square odd-sided weight stencil (kernels_regular.py:327-356)."""

    weights: np.ndarray

    def __post_init__(self) -> None:
        w = np.asarray(self.weights)
        if w.ndim != 2 or w.shape[0] != w.shape[1] or w.shape[0] % 2 == 0:
            raise ValueError("kernel must be square with odd side")
        if not np.isfinite(w).all():
            raise ValueError("kernel weights must be finite")

    @property
    def radius(self) -> int:
        return self.weights.shape[0] // 2

    @classmethod
    def delta(cls, radius: int) -> "FilterKernel":
        w = np.zeros((2 * radius + 1, 2 * radius + 1))
        w[radius, radius] = 1.0
        return cls(w)

    @classmethod
    def gaussian(cls, radius: int, sigma: float | None = None) -> "FilterKernel":
        sigma = sigma or max(radius / 2.0, 0.5)
        ax = np.arange(-radius, radius + 1, dtype=np.float64)
        g = np.exp(-(ax[:, None] ** 2 + ax[None, :] ** 2) / (2.0 * sigma**2))
        return cls(g / g.sum())


def convolve_rows(pixels: Any, kernel: FilterKernel, row0: int, row1: int, workers: int = 1,
                  out: np.ndarray | None = None) -> np.ndarray:
    """Host (DeviceA) body, the reference arithmetic (:359-381) in native code
    (hb_host_conv_rows on `workers` threads): correlation of rows [row0, row1)
    with clamp-to-edge borders, one weighted plane added per non-zero tap in
    row-major order; float64 rows."""
    arr = to_host(pixels)
    if arr.dtype not in (np.uint8, np.float64):
        arr = arr.astype(np.float64)
    arr = np.ascontiguousarray(arr)
    height, width = arr.shape
    out = _host_rows_out(out, row1 - row0, width)
    if row1 <= row0:
        return out
    if not 0 <= row0 and row1 <= height:
        raise ValueError("bad row range")
    w = np.ascontiguousarray(kernel.weights, dtype=np.float64)
    _lib.call("hb_host_conv_rows", vp(arr.ctypes.data), _lib.DTYPE_CODES["u1" if arr.dtype == np.uint8 else "f8"],
              height, width, kernel.radius, vp(w.ctypes.data), row0, row1, vp(out.ctypes.data), workers)
    return out


def _device_table(owner: Any, key: str, table: np.ndarray, device: Any) -> Any:
    """A float64 CUDA copy of a small weight table (LUT / stencil), cached on
    its owner per device so repeated device-resident calls neither re-upload
    it nor synchronise (and stay CUDA-graph capturable).  The cached host copy
    is compared on every call, so an owner whose array was changed in place
    gets a fresh upload."""
    import torch

    host = np.ascontiguousarray(table, dtype=np.float64)
    cache = owner.__dict__.get("_device_tables")
    if cache is None:
        cache = {}
        object.__setattr__(owner, "_device_tables", cache)
    slot = (key, str(device))
    hit = cache.get(slot)
    if hit is not None and np.array_equal(hit[0], host):
        return hit[1]
    snap = host.copy()
    dev = torch.from_numpy(snap.copy()).to(device)
    cache[slot] = (snap, dev)
    return dev


def gpu_convolve_rows(pixels: Any, kernel: FilterKernel, row0: int, row1: int, out: Any = None,
                      *, out_dtype: Any = np.float64, asynchronous: bool = False,
                      arithmetic: str = "fp64") -> Any:
    """DeviceB body (hb_convolve): rows [row0, row1) on the GPU, bit-identical
    to `convolve_rows` for fp64 output.  uint8 and float64 pixels go to the
    kernel as they are; other dtypes are widened to float64 first (exactly
    what `astype(np.float64)` does in the reference).  Host pixels → numpy
    result; CUDA pixels → result tensor.  arithmetic="fp32": fp32 taps with
    FMA, within 1e-5 relative of the fp64 result."""
    _lib.load()
    code = 64 if np.dtype(out_dtype) == np.float64 else 32
    if arithmetic not in ("fp64", "fp32"):
        raise ValueError(f"arithmetic must be 'fp64' or 'fp32', got {arithmetic!r}")
    math_flag = _lib.HB_FP32_ARITH if arithmetic == "fp32" else 0
    height, width = int(pixels.shape[0]), int(pixels.shape[1])
    if not 0 <= row0 <= row1 <= height:
        raise ValueError("bad row range")
    if row1 > row0:
        require_gpu()
    w = np.ascontiguousarray(kernel.weights, dtype=np.float64)
    if is_device_array(pixels):
        import torch

        if pixels.dtype not in (torch.uint8, torch.float64):
            pixels = pixels.to(torch.float64)
        pixels = pixels.contiguous()
        tdt = torch.float64 if code == 64 else torch.float32
        if out is None:
            out = torch.empty((row1 - row0, width), dtype=tdt, device=pixels.device)
        if row1 == row0:
            return out
        wt = _device_table(kernel, "weights", w, pixels.device)
        in_code = _lib.DTYPE_CODES["u1" if pixels.dtype == torch.uint8 else "f8"]
        flags = _lib.HB_DEVICE_PTRS | (_lib.HB_ASYNC if asynchronous else 0) | math_flag
        if bool(np.all(w != 0.0)):
            flags |= _lib.HB_TAPS_DENSE  # the host weights tell: no read-back, no host wait
        _lib.call("hb_convolve", vp(pixels.data_ptr()), in_code, height, width, kernel.radius, vp(wt.data_ptr()),
                  row0, row1, vp(out.data_ptr()), code, flags, current_stream_handle(pixels))
        return out
    arr = np.asarray(pixels)
    if arr.dtype not in (np.uint8, np.float64):
        arr = arr.astype(np.float64)
    img = buf(arr)
    if out is None:
        out = host_empty((row1 - row0, width), np.float64 if code == 64 else np.float32)
    if row1 == row0:
        return out
    _lib.call("hb_convolve", vp(img.ptr), img.code, height, width, kernel.radius, vp(w.ctypes.data),
              row0, row1, vp(out.ctypes.data), code, math_flag, current_stream_handle())
    return out


class ConvolutionWorkload(_StripOutput):
    """Horizontal strip split at floor(f·H); halo rows are read from the
    shared source image (kernels_regular.py:384-405).  DeviceA: native host
    threads; DeviceB: the GPU tile kernel over the GPU group (floor(k·n/G)
    strips); both write into one output image (_StripOutput)."""

    name = "conv"
    unit = "neighbor accumulations"

    def __init__(self, image: Image, kernel: FilterKernel, arithmetic: str = "fp64"):
        self.image = image
        self.kernel = kernel
        self.arithmetic = arithmetic  # "fp32": the GPU share's taps in fp32 (within 1e-5 relative)
        self._per_row = image.width * (2 * kernel.radius + 1) ** 2

    def partition(self, fraction_a: float):
        split = int(math.floor(fraction_a * self.image.height))
        self._new_output(self.image.height, self.image.width)
        return (0, split), (split, self.image.height)

    def work_units(self, part) -> float:
        return float((part[1] - part[0]) * self._per_row)

    def run_part(self, device: Device, part) -> np.ndarray:
        strip = self._strip(part)
        if device.id is DeviceId.B:
            ar = self.arithmetic
            if strip is not None:
                return gpu_convolve_rows(self.image.pixels, self.kernel, part[0], part[1], out=strip, arithmetic=ar)
            return sharding.run_sharded_rows(
                part[0], part[1], lambda a, b: gpu_convolve_rows(self.image.pixels, self.kernel, a, b, arithmetic=ar)
            )
        return convolve_rows(self.image.pixels, self.kernel, part[0], part[1], device.worker_count, out=strip)


def hybrid_convolve(image: Image, kernel: FilterKernel, platform: Platform,
                    share: WorkShare | None = None, *, arithmetic: str = "fp64") -> Image:
    """kernels_regular.py:408-414 (+ `arithmetic`, this package's fp32 mode)."""
    workload = ConvolutionWorkload(image, kernel, arithmetic)
    result, _ = run_workshared(platform, workload, share or formula_share(platform), baselines=False)
    return result


# --------------------------------------------------------------------------
# bilateral filter (kernels_regular.py:421-520)


@dataclass(frozen=True)
class BilateralLut:
    """Gaussian tables: spatial weight per stencil offset (row-major), range
    weight per absolute intensity difference (:421-444)."""

    spatial_weights: np.ndarray
    range_weights: np.ndarray
    sigma_s: float
    sigma_r: float
    radius: int

    def __post_init__(self) -> None:
        side = 2 * self.radius + 1
        if self.spatial_weights.shape != (side * side,):
            raise ValueError("spatial table must have (2r+1)^2 entries")
        if self.range_weights.shape != (256,):
            raise ValueError("range table must have 256 entries")
        for table in (self.spatial_weights, self.range_weights):
            if not ((table > 0) & (table <= 1.0)).all():
                raise ValueError("lut weights must lie in (0, 1]")

    @property
    def entry_count(self) -> int:
        return self.spatial_weights.size + self.range_weights.size


def build_bilateral_lut(radius: int, sigma_s: float, sigma_r: float) -> BilateralLut:
    """spatial[d] = exp(-|offset|^2 / 2σs²), range[k] = exp(-k² / 2σr²) (:447-458)."""
    if radius < 0:
        raise ValueError("radius must be >= 0")
    if not (sigma_s > 0 and sigma_r > 0):
        raise ValueError("sigmas must be > 0")
    off = np.arange(-radius, radius + 1, dtype=np.float64)
    d2 = off[:, None] ** 2 + off[None, :] ** 2
    spatial = np.exp(-d2 / (2.0 * sigma_s**2)).ravel()
    k = np.arange(256, dtype=np.float64)
    return BilateralLut(spatial, np.exp(-(k**2) / (2.0 * sigma_r**2)), sigma_s, sigma_r, radius)


def bilateral_rows(pixels: Any, lut: BilateralLut, row0: int, row1: int, workers: int = 1,
                   out: np.ndarray | None = None) -> np.ndarray:
    """Host (DeviceA) body, the reference arithmetic (:461-486) in native code
    (hb_host_bilateral on `workers` threads): for each tap in row-major order
    w = spatial·range[|nb-c|], num += w·nb, den += w; clamp to edge; returns
    num/den as float64 rows [row0, row1)."""
    pix = np.ascontiguousarray(to_host(pixels), dtype=np.uint8)
    height, width = pix.shape
    out = _host_rows_out(out, row1 - row0, width)
    if row1 <= row0:
        return out
    if not 0 <= row0 and row1 <= height:
        raise ValueError("bad row range")
    sp = np.ascontiguousarray(lut.spatial_weights, dtype=np.float64)
    rg = np.ascontiguousarray(lut.range_weights, dtype=np.float64)
    _lib.call("hb_host_bilateral", vp(pix.ctypes.data), height, width, lut.radius, vp(sp.ctypes.data),
              vp(rg.ctypes.data), row0, row1, vp(out.ctypes.data), workers)
    return out


def gpu_bilateral_rows(pixels: Any, lut: BilateralLut, row0: int, row1: int, out: Any = None,
                       *, out_dtype: Any = np.float64, asynchronous: bool = False,
                       arithmetic: str = "fp64") -> Any:
    """DeviceB body (hb_bilateral_u8): rows [row0, row1) on the GPU, bit-identical
    to `bilateral_rows` for fp64 output.  Host pixels → numpy result; CUDA
    pixels (uint8 tensor) → result tensor (the LUT tables are staged per call).
    arithmetic="fp32": taps in fp32 with FMA — within 1e-5 relative of the
    fp64 result (north_star's filter tolerance), about twice as fast."""
    _lib.load()
    code = 64 if np.dtype(out_dtype) == np.float64 else 32
    if arithmetic not in ("fp64", "fp32"):
        raise ValueError(f"arithmetic must be 'fp64' or 'fp32', got {arithmetic!r}")
    math_flag = _lib.HB_FP32_ARITH if arithmetic == "fp32" else 0
    height, width = int(pixels.shape[0]), int(pixels.shape[1])
    if not 0 <= row0 <= row1 <= height:
        raise ValueError("bad row range")
    if row1 > row0:
        require_gpu()
    if is_device_array(pixels):
        import torch

        # the host path's cast (np.ascontiguousarray(..., dtype=uint8)); the
        # kernel reads raw contiguous uint8 rows
        pixels = pixels.to(torch.uint8).contiguous()
        tdt = torch.float64 if code == 64 else torch.float32
        if out is None:
            out = torch.empty((row1 - row0, width), dtype=tdt, device=pixels.device)
        if row1 == row0:
            return out
        sp = _device_table(lut, "spatial", lut.spatial_weights, pixels.device)
        rg = _device_table(lut, "range", lut.range_weights, pixels.device)
        flags = _lib.HB_DEVICE_PTRS | (_lib.HB_ASYNC if asynchronous else 0) | math_flag
        _lib.call("hb_bilateral_u8", vp(pixels.data_ptr()), height, width, lut.radius, vp(sp.data_ptr()),
                  vp(rg.data_ptr()), row0, row1, vp(out.data_ptr()), code, flags, current_stream_handle(pixels))
        return out
    img = buf(pixels, np.uint8)
    if out is None:
        out = host_empty((row1 - row0, width), np.float64 if code == 64 else np.float32)
    if row1 == row0:
        return out
    sp = np.ascontiguousarray(lut.spatial_weights, dtype=np.float64)
    rg = np.ascontiguousarray(lut.range_weights, dtype=np.float64)
    _lib.call("hb_bilateral_u8", vp(img.ptr), height, width, lut.radius, vp(sp.ctypes.data),
              vp(rg.ctypes.data), row0, row1, vp(out.ctypes.data), code, math_flag, current_stream_handle())
    return out


class BilateralApplyWorkload(_StripOutput):
    """Row strips split at floor(f·H) (:489-511).  DeviceA: numpy rows;
    DeviceB: the GPU tile kernel, its strip split again over the GPU group
    (floor(k·n/G)) and gathered; the merge stacks the strips."""

    name = "bilat"
    unit = "neighbor accumulations"

    def __init__(self, image: Image, lut: BilateralLut, arithmetic: str = "fp64"):
        self.image = image
        self.lut = lut
        self.arithmetic = arithmetic  # "fp32": the GPU share's taps in fp32 (within 1e-5 relative)
        self._per_row = image.width * (2 * lut.radius + 1) ** 2

    def partition(self, fraction_a: float):
        split = int(math.floor(fraction_a * self.image.height))
        self._new_output(self.image.height, self.image.width)
        return (0, split), (split, self.image.height)

    def work_units(self, part) -> float:
        return float((part[1] - part[0]) * self._per_row)

    def run_part(self, device: Device, part) -> np.ndarray:
        strip = self._strip(part)
        if device.id is DeviceId.B:
            ar = self.arithmetic
            if strip is not None:
                return gpu_bilateral_rows(self.image.pixels, self.lut, part[0], part[1], out=strip, arithmetic=ar)
            return sharding.run_sharded_rows(
                part[0], part[1], lambda a, b: gpu_bilateral_rows(self.image.pixels, self.lut, a, b, arithmetic=ar)
            )
        return bilateral_rows(self.image.pixels, self.lut, part[0], part[1], device.worker_count, out=strip)


def hybrid_bilateral(image: Image, lut: BilateralLut, platform: Platform, share: WorkShare | None = None,
                     *, arithmetic: str = "fp64") -> Image:
    """kernels_regular.py:514-520 (+ `arithmetic`, this package's fp32 mode)."""
    workload = BilateralApplyWorkload(image, lut, arithmetic)
    result, _ = run_workshared(platform, workload, share or formula_share(platform), baselines=False)
    return result
