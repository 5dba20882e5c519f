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
