"""Regular hot-path kernels behind the reference's own entry points
(hybridbench/kernels_regular.py): histogram, sort, bilateral filter.

Each workload keeps the reference's Partitionable protocol and names.
`run_part(DeviceA, …)` computes the host share with numpy on the host
cores; `run_part(DeviceB, …)` is the GPU share, one libhb200 call (sharded
over the active GPU group, see sharding.py).  Inputs may be numpy arrays
(host; staged inside the C call) or CUDA tensors (device-resident).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Any, Sequence

import numpy as np

from . import _lib, sharding
from .gpu import buf, current_stream_handle, flags_for, is_device_array, require_gpu, to_host, vp
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
    if b.code == 0:
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
        host = to_host(part)
        counts = np.zeros(self.bin_count, dtype=np.int64)
        edges = np.linspace(0, host.size, device.worker_count + 1).astype(np.int64)
        for lo, hi in zip(edges[:-1], edges[1:]):
            counts += np.bincount(host[lo:hi], minlength=self.bin_count)
        return counts

    def merge(self, partials: Sequence[np.ndarray]) -> HistogramResult:
        total = np.zeros(self.bin_count, dtype=np.int64)
        for p in partials:
            total += p
        return HistogramResult(total, self.bin_count)


def hybrid_histogram(
    data: Any, bin_count: int, platform: Platform, share: WorkShare | None = None
) -> HistogramResult:
    """kernels_regular.py:163-169: work-shared histogram, no baselines."""
    workload = HistogramWorkload(data, bin_count)
    result, _ = run_workshared(platform, workload, share or formula_share(platform), baselines=False)
    return result
