"""Pageable host <-> device copy costs through the C ABI (hb_buf_upload /
hb_buf_download: pinned double-buffer staging + threaded memcpy), 1 GiB:
upload from a touched pageable array, download into a fresh np.empty (first
touch inside the copy) vs into a touched array, and the first-touch rate
itself.  Also prints the host's transparent-hugepage settings."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1303_2171_b200 import _lib

for f in ("enabled", "defrag"):
    try:
        print(f"THP {f}:", Path(f"/sys/kernel/mm/transparent_hugepage/{f}").read_text().strip())
    except OSError as e:
        print("THP", f, e)
n = 1 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
src = np.ones(n, dtype=np.uint8)
vp = ctypes.c_void_p


def t(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - a)
    return min(out), float(np.median(out))


def up():
    _lib.call("hb_buf_upload", vp(d.data_ptr()), vp(src.ctypes.data), n, 0, vp(0))


touched = np.zeros(n, dtype=np.uint8)


def down_touched():
    _lib.call("hb_buf_download", vp(touched.ctypes.data), vp(d.data_ptr()), n, 0, vp(0))


def down_fresh():
    r = np.empty(n, dtype=np.uint8)
    _lib.call("hb_buf_download", vp(r.ctypes.data), vp(d.data_ptr()), n, 0, vp(0))


def touch_fresh():
    r = np.empty(n, dtype=np.uint8)
    r[::4096] = 1


def fill_fresh():
    r = np.empty(n, dtype=np.uint8)
    r.fill(1)


def down_fresh_4k():
    from numpy._core import multiarray as ma

    prev = ma._set_madvise_hugepage(False)  # numpy madvises large arrays MADV_HUGEPAGE by default
    try:
        r = np.empty(n, dtype=np.uint8)
    finally:
        ma._set_madvise_hugepage(prev)
    _lib.call("hb_buf_download", vp(r.ctypes.data), vp(d.data_ptr()), n, 0, vp(0))


for name, fn in [("upload pageable (touched)", up), ("download into touched", down_touched),
                 ("download into fresh np.empty, 4 KB pages", down_fresh_4k),
                 ("download into fresh np.empty", down_fresh), ("first touch only (1 byte/page, 1 thread)", touch_fresh),
                 ("fill fresh np.empty (1 thread)", fill_fresh)]:
    mn, md = t(fn)
    print(f"{name:45s} min {mn * 1e3:7.2f} ms  median {md * 1e3:7.2f} ms  -> {n / md / 1e9:6.1f} GB/s", flush=True)
