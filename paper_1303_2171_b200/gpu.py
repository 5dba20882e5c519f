"""Host-side plumbing between numpy / torch arrays and the C ABI.

A *buffer* handed to a `hb_*` call is either a host array (numpy; the
library stages it through device memory inside the call) or a CUDA tensor
(torch, device-resident; the call passes `HB_DEVICE_PTRS` and works in place
on the caller's stream).  PyTorch is only plumbing here — device memory,
streams and `torch.distributed`; every computation is a libhb200 kernel.
"""

from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass
from typing import Any

import numpy as np

from . import _lib

try:  # torch is optional for host-array use; required for device-resident use
    import torch
except Exception:  # pragma: no cover - torch is in the image
    torch = None  # type: ignore[assignment]


def is_device_array(x: Any) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def require_gpu() -> None:
    """Fail loudly when the GPU share cannot run (no silent CPU fallback)."""
    _lib.load()
    if _lib.device_count() < 1:
        from .errors import HybridBenchError

        raise HybridBenchError("no CUDA device visible: the DeviceB (GPU) share cannot run")


def inherit_device(fn: Any) -> Any:
    """Wrap `fn` for another thread so that it runs on the CALLING thread's
    CUDA device.  The CUDA runtime's current device is per host thread and a
    new thread starts on device 0, so without this the run_part threads of a
    rank bound to cuda:k (torchrun, one process per GPU) would allocate,
    copy and launch on GPU 0."""
    dev = None
    if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
        dev = torch.cuda.current_device()
    if dev is None:
        return fn

    def run(*args: Any, **kwargs: Any) -> Any:
        if torch.cuda.current_device() != dev:
            torch.cuda.set_device(dev)
        return fn(*args, **kwargs)

    return run


def current_stream_handle(x: Any = None) -> int:
    """cudaStream_t of torch's current stream (0 = legacy default stream)."""
    if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
        dev = x.device if is_device_array(x) else None
        return int(torch.cuda.current_stream(dev).cuda_stream)
    return 0


_TORCH_TO_NP = {}
if torch is not None:
    _TORCH_TO_NP = {
        torch.uint8: np.dtype(np.uint8),
        torch.int8: np.dtype(np.int8),
        torch.int16: np.dtype(np.int16),
        torch.int32: np.dtype(np.int32),
        torch.int64: np.dtype(np.int64),
        torch.float32: np.dtype(np.float32),
        torch.float64: np.dtype(np.float64),
    }
    for _name in ("uint16", "uint32", "uint64"):
        if hasattr(torch, _name):
            _TORCH_TO_NP[getattr(torch, _name)] = np.dtype(_name)


@dataclass
class Buf:
    """A raw view of an array for the C ABI."""

    ptr: int
    size: int  # elements
    dtype: np.dtype
    device: bool
    owner: Any  # keeps the memory alive for the duration of the call

    @property
    def nbytes(self) -> int:
        return self.size * self.dtype.itemsize

    @property
    def code(self) -> int:
        return _lib.DTYPE_CODES[self.dtype.str[1:]] if self.dtype.str[1:] in _lib.DTYPE_CODES else 0


def buf(x: Any, dtype: Any = None) -> Buf:
    """View `x` (numpy array or CUDA tensor) as a C-ABI buffer.  Host arrays
    are made C-contiguous (and cast to `dtype` when given); device tensors
    must already be contiguous and of the right dtype."""
    if is_device_array(x):
        if not x.is_contiguous():
            x = x.contiguous()
        dt = _TORCH_TO_NP.get(x.dtype)
        if dt is None:
            raise TypeError(f"unsupported tensor dtype {x.dtype}")
        if dtype is not None and np.dtype(dtype) != dt:
            raise TypeError(f"expected a {np.dtype(dtype)} tensor, got {x.dtype}")
        return Buf(x.data_ptr(), x.numel(), dt, True, x)
    arr = np.asarray(x)
    if dtype is not None and arr.dtype != np.dtype(dtype):
        arr = arr.astype(dtype)
    arr = np.ascontiguousarray(arr)
    return Buf(arr.ctypes.data if arr.size else 0, arr.size, arr.dtype, False, arr)


def out_like(device: bool, shape: Any, dtype: Any, ref: Any = None) -> Any:
    """Allocate an output on the same side as the input."""
    if device:
        return torch.empty(shape, dtype=_np_to_torch(np.dtype(dtype)), device=ref.device if ref is not None else "cuda")
    return np.empty(shape, dtype=dtype)


PINNED_MIN_BYTES = 4 << 20
PINNED_MAX_BYTES = 8 << 30
PINNED_POOL_CAP = 8 << 30  # page-locked result blocks the library may make torch cache


class _ResultPool:
    """Bookkeeping of large host results by power-of-two size class (torch's
    caching host allocator rounds block sizes up to powers of two): which
    results the caller still holds, how many the caller has dropped, and how
    many of the library's page-locked result blocks are back in torch's
    cache, free to be handed out again."""

    def __init__(self):
        import itertools
        import threading

        self.lock = threading.Lock()
        self.pending: Any = __import__("collections").deque()  # released keys not yet booked
        self.keys = itertools.count()
        self.live: dict[int, tuple[int, Any, bool]] = {}  # key -> (class, scope token, pinned)
        self.dropped: dict[int, int] = {}  # class -> results the caller let go of
        self.free: dict[int, int] = {}     # class -> our page-locked blocks back in torch's cache
        self.pinned_bytes = 0              # page-locked result blocks ever made (torch keeps them)

    def released(self, key: int) -> None:
        # finalizer: may run inside any allocation, even one made while this
        # thread holds `lock` (a garbage collection there), so it only queues
        # the key (deque.append is atomic); book() settles it under the lock
        self.pending.append(key)

    def book(self) -> None:
        """Settle queued releases (caller holds `lock`)."""
        while self.pending:
            c, _, pinned = self.live.pop(self.pending.popleft())
            self.dropped[c] = self.dropped.get(c, 0) + 1
            if pinned:
                self.free[c] = self.free.get(c, 0) + 1


_pool = _ResultPool()
_scope = __import__("threading").local()


@contextlib.contextmanager
def result_scope():
    """Results allocated inside one scope belong to one API call (e.g. the
    sorted keys and the payload of gpu_sort): one result of the call being
    live does not keep the next from being page-locked."""
    prev = getattr(_scope, "token", None)
    _scope.token = object()
    try:
        yield
    finally:
        _scope.token = prev


def host_empty(shape: Any, dtype: Any = np.float64) -> np.ndarray:
    """An uninitialised host array for a result the GPU writes back.

    Costs on the B200 box (scripts/prof_pageable.py, per GiB): the D2H into
    page-locked memory is one DMA (~19 ms); into a fresh pageable array it
    pays the first-touch zeroing of the pages (~50 ms); pinning FRESH memory
    (cudaHostAlloc) costs ~450 ms — more than it can save in one call.  So a
    large result is page-locked only when that is free or pays back:
      * one of the library's earlier page-locked results of the same size
        class has been dropped (its block sits in torch's host cache): reuse;
      * else, the caller has dropped an earlier result of this class and
        holds none now (a loop that drops each result): pin once — every
        later call reuses the block;
      * else (a first call, or a caller that keeps its results): pageable.
    Results of one API call (`result_scope`) do not hold each other back.
    Small results, results above PINNED_MAX_BYTES and hosts without CUDA are
    plain np.empty."""
    import weakref

    dt = np.dtype(dtype)
    shape = (int(shape),) if np.ndim(shape) == 0 else tuple(int(d) for d in shape)
    nbytes = int(np.prod(shape, dtype=np.int64)) * dt.itemsize
    if not (torch is not None and PINNED_MIN_BYTES <= nbytes <= PINNED_MAX_BYTES and dt in _TORCH_TO_NP.values()
            and torch.cuda.is_available()):
        return np.empty(shape, dtype=dt)
    c = 1 << (nbytes - 1).bit_length()
    token = getattr(_scope, "token", None)
    with _pool.lock:
        _pool.book()
        held = any(cc == c and not (token is not None and t is token) for cc, t, _ in _pool.live.values())
        if _pool.free.get(c, 0) > 0:
            _pool.free[c] -= 1
            pin = True
        elif _pool.dropped.get(c, 0) > 0 and not held and _pool.pinned_bytes + c <= PINNED_POOL_CAP:
            _pool.pinned_bytes += c
            pin = True
        else:
            pin = False
        key = next(_pool.keys)
        _pool.live[key] = (c, token, pin)
    arr = None
    if pin:
        try:
            arr = torch.empty(shape, dtype=_np_to_torch(dt), pin_memory=True).numpy()
        except RuntimeError:  # pinned memory exhausted: pageable result
            with _pool.lock:
                _pool.book()
                _pool.live[key] = (c, token, False)
    if arr is None:
        arr = np.empty(shape, dtype=dt)
    weakref.finalize(arr, _pool.released, key)
    return arr


def _np_to_torch(dt: np.dtype):
    for k, v in _TORCH_TO_NP.items():
        if v == dt:
            return k
    raise TypeError(f"no torch dtype for {dt}")


def flags_for(*bufs: Buf, asynchronous: bool = False) -> int:
    """HB_DEVICE_PTRS when every buffer is device memory; mixing is refused."""
    kinds = {b.device for b in bufs if b.size or b.ptr}
    if len(kinds) > 1:
        raise ValueError("mixing host arrays and CUDA tensors in one call is not supported")
    dev = kinds == {True}
    f = _lib.HB_DEVICE_PTRS if dev else 0
    if asynchronous and dev:
        f |= _lib.HB_ASYNC
    return f


def to_host(x: Any) -> np.ndarray:
    if is_device_array(x):
        return x.cpu().numpy()
    return np.asarray(x)


def vp(ptr: int) -> ctypes.c_void_p:
    return ctypes.c_void_p(ptr)
