"""The C-ABI library loads here (no GPU) and exports every entry point the
header declares; the Python binding covers all of them.  CPU only."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_1303_2171_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "hb200.h"


def declared() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"^(?:int|const char\*)\s+(hb_\w+)\s*\(", text, flags=re.M))


def test_header_declares_entry_points():
    names = declared()
    assert {"hb_hist", "hb_last_error", "hb_gen_splitmix"} <= names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in sorted(declared()) if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(_lib.exported_symbols()) == declared()


def test_runtime_calls_without_gpu():
    lib = _lib.load()
    assert lib.hb_version() >= 1
    assert _lib.device_count() >= 0


def test_argument_errors_map_to_value_error():
    # argument validation happens before any device work
    with pytest.raises(ValueError):
        _lib.call("hb_hist", None, 99, 10, 256, None, 0, None)
    with pytest.raises(ValueError):
        _lib.call("hb_hist", None, 1, 10, 0, None, 0, None)


@pytest.mark.gpu
def test_torch_free_device_resident_round_trip():
    """The reference-side binding without a GPU framework: allocate, upload,
    run hb_hist on device buffers, download, free — through ctypes only."""
    import numpy as np

    lib = _lib.load()
    assert lib.hb_set_device(0) == 0
    data = (np.arange(1 << 20, dtype=np.int64) * 2654435761 % 251).astype(np.uint8)
    d_in, d_out, stream = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    _lib.call("hb_stream_create", ctypes.byref(stream))
    _lib.call("hb_buf_alloc", data.nbytes, ctypes.byref(d_in))
    _lib.call("hb_buf_alloc", 256 * 8, ctypes.byref(d_out))
    try:
        _lib.call("hb_buf_upload", d_in, data.ctypes.data, data.nbytes, 0, stream)
        _lib.call("hb_hist", d_in, _lib.DTYPE_CODES["u1"], data.size, 256, d_out, _lib.HB_DEVICE_PTRS, stream)
        got = np.zeros(256, dtype=np.uint64)
        _lib.call("hb_buf_download", got.ctypes.data, d_out, got.nbytes, 0, stream)
        assert np.array_equal(got.astype(np.int64), np.bincount(data, minlength=256))
    finally:
        _lib.call("hb_buf_free", d_in)
        _lib.call("hb_buf_free", d_out)
        _lib.call("hb_stream_destroy", stream)
