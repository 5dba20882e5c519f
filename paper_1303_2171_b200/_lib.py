"""ctypes binding of libhb200.so (the C ABI declared in include/hb200.h).

`ctypes.CDLL` releases the GIL for the duration of every call, so the two
`run_workshared` threads (reference worksharing.py:317-320) really overlap:
the host share keeps running numpy while the GPU share waits on its stream.

The library is built in-tree (`__graft_entry__.build()` → csrc/Makefile);
there is no fallback: if it is missing or cannot be loaded, every GPU entry
point raises `HybridBenchError` instead of silently computing on the CPU.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import HybridBenchError, StructuralError

LIB_PATH = Path(__file__).resolve().parent / "libhb200.so"

HB_OK, HB_EINVAL, HB_ESTRUCT, HB_ECUDA, HB_ENOMEM, HB_ENOSYS = range(6)
HB_DEVICE_PTRS = 1
HB_ASYNC = 2
HB_ACCUMULATE = 4
HB_SORT_BALLOT = 8
HB_FP32_ARITH = 16
HB_TAPS_DENSE = 32

HB_GEN_RAW, HB_GEN_LOW8, HB_GEN_HI32, HB_GEN_MOD = range(4)
HB_SPMV_SEQ, HB_SPMV_WARP, HB_SPMV_MERGE = 0, 1, 2

# numpy dtype.str (sans byte order) -> element code of include/hb200.h
DTYPE_CODES = {"u1": 1, "i1": 2, "u2": 3, "i2": 4, "u4": 5, "i4": 6, "u8": 7, "i8": 8, "f8": 9}

_c = ctypes
_vp, _i32, _i64, _u64 = _c.c_void_p, _c.c_int32, _c.c_int64, _c.c_uint64
_int = _c.c_int

# name -> argtypes; every function returns int (status)
_SIGNATURES: dict[str, list] = {
    "hb_version": [],
    "hb_device_count": [_c.POINTER(_int)],
    "hb_sm_count": [_c.POINTER(_int)],
    "hb_stream_sync": [_vp],
    "hb_trim": [],
    "hb_set_device": [_int],
    "hb_buf_alloc": [_c.c_size_t, _c.POINTER(_vp)],
    "hb_buf_free": [_vp],
    "hb_buf_upload": [_vp, _vp, _c.c_size_t, _int, _vp],
    "hb_buf_download": [_vp, _vp, _c.c_size_t, _int, _vp],
    "hb_stream_create": [_c.POINTER(_vp)],
    "hb_stream_destroy": [_vp],
    "hb_gen_splitmix": [_u64, _u64, _i64, _int, _u64, _vp, _vp],
    "hb_hist": [_vp, _int, _i64, _i32, _vp, _int, _vp],
    "hb_spmv_csr": [_vp, _int, _vp, _int, _vp, _i64, _i64, _i64, _vp, _vp, _int, _vp, _int, _int, _vp],
    "hb_csr_validate": [_vp, _int, _vp, _int, _i64, _i64, _i64, _vp, _int, _vp],
    "hb_spmv_preprocess": [_vp, _int, _vp, _int, _vp, _i64, _vp, _int, _vp, _vp, _vp, _int, _vp],
    "hb_bilateral_u8": [_vp, _i32, _i32, _i32, _vp, _vp, _i32, _i32, _vp, _int, _int, _vp],
    "hb_convolve": [_vp, _int, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _int, _int, _vp],
    "hb_host_hist": [_vp, _int, _i64, _i32, _vp, _int],
    "hb_host_spmv_rows": [_vp, _int, _vp, _int, _vp, _i64, _i64, _vp, _vp, _int, _vp, _int],
    "hb_host_conv_rows": [_vp, _int, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _int],
    "hb_host_bilateral": [_vp, _i32, _i32, _i32, _vp, _vp, _i32, _i32, _vp, _int],
    "hb_sort": [_vp, _vp, _int, _vp, _vp, _i64, _vp, _int, _vp],
    "hb_sort_bounds": [_vp, _int, _vp, _i64, _vp, _vp, _i32, _vp, _int, _vp],
    "hb_list_rank": [_vp, _int, _i64, _i64, _vp, _int, _vp],
    "hb_link_order": [_vp, _i64, _vp, _int, _int, _vp],
    "hb_list_fis_stats": [_vp, _int, _i64, _i64, _u64, _i32, _vp, _i32, _vp, _int, _vp],
    "hb_gen_csr": [_i64, _i64, _i64, _u64, _u64, _u64, _vp, _int, _vp, _int, _vp, _i64, _vp, _int, _vp],
    "hb_spmv_sell_build": [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _int, _vp],
    "hb_spmv_sell": [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _int, _vp, _int, _vp],
    "hb_partition_nnz": [_vp, _int, _i64, _i64, _i32, _vp, _int, _vp],
    "hb_scatter_perm": [_vp, _i64, _int, _vp, _int, _vp, _int, _vp],
    "hb_merge_runs": [_vp, _int, _vp, _i64, _vp, _i32, _vp, _vp, _int, _vp],
    "hb_lr_layout": [_i64, _i64, _vp, _vp],
    "hb_lr_walk_part": [_vp, _int, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _int, _vp],
    "hb_lr_finish_part": [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _int, _vp],
    "hb_lr_finish_part32": [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _int, _vp],
    "hb_widen_i32": [_vp, _i64, _vp, _int, _vp],
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def exported_symbols() -> list[str]:
    """Every entry point the Python layer binds (all declared in hb200.h)."""
    return sorted(_SIGNATURES) + ["hb_last_error"]


def load() -> ctypes.CDLL:
    """Load libhb200.so once; raise loudly when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = Path(os.environ.get("HB200_LIB", LIB_PATH))
        if not path.exists():
            raise HybridBenchError(
                f"libhb200.so not found at {path}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the GPU share)"
            )
        try:
            lib = ctypes.CDLL(str(path))
        except OSError as exc:
            raise HybridBenchError(f"cannot load {path}: {exc}") from exc
        for name, argtypes in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _int
        lib.hb_last_error.argtypes = []
        lib.hb_last_error.restype = _c.c_char_p
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().hb_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, what: str) -> None:
    """Map a C-ABI status onto the reference exception hierarchy."""
    if rc == HB_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == HB_EINVAL:
        raise ValueError(msg)
    if rc == HB_ESTRUCT:
        raise StructuralError(msg)
    raise HybridBenchError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def device_count() -> int:
    n = _int(0)
    call("hb_device_count", _c.byref(n))
    return n.value


def sm_count() -> int:
    n = _int(0)
    call("hb_sm_count", _c.byref(n))
    return n.value
