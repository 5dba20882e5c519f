"""The reference side of bench.py: the UNMODIFIED reference package
(`hybridbench`, installed under baseline/_ref with
`pip install --no-index --no-deps --target baseline/_ref <copy of /root/reference/pkg>`)
timed through its own public entry points on the host cores.

Used twice: `bench.py --impl reference` (the reference arm: inputs made
here with the threaded numpy splitmix64 below or the reference's own
generators — nothing imports torch, libhb200 or the product package, so
that arm loads no native code of this repository), and bench.py's
`cpu_baseline` legs (the same reference calls on host copies of the very
inputs the GPU arm ran on).  When baseline/_ref is absent (a fresh
checkout) the numpy restatement under oracle/ is timed instead and the
line says `kind: "port"`.

Each leg returns (fn, units, sample, cores, kind, same_config): `fn()` runs
one step of the reference on its input; `units / t` is the metric.
"""

from __future__ import annotations

import os
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
REF_DIR = ROOT / "baseline" / "_ref"

_G = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def reference_available() -> bool:
    return (REF_DIR / "hybridbench" / "__init__.py").exists()


def import_reference():
    """The installed reference package (baseline/_ref), never /root/reference."""
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import hybridbench  # noqa: F401

    return hybridbench


def splitmix_low8(seed: int, n: int, k0: int = 0, threads: int | None = None) -> np.ndarray:
    """uint8 draws k0+1 .. k0+n of splitmix64(seed) & 255 — the reference's
    gen_hist_data / gen_image values (datasets.py:33-34, 104-106,
    rng.py:45-51) — computed in 4 Mi-element chunks on a thread pool (numpy
    releases the GIL in its ufuncs)."""
    out = np.empty(n, dtype=np.uint8)
    chunk = 1 << 22
    seed64 = np.uint64(seed & ((1 << 64) - 1))

    def fill(lo: int) -> None:
        hi = min(n, lo + chunk)
        k = np.arange(k0 + lo + 1, k0 + hi + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = seed64 + k * _G
            z ^= z >> np.uint64(30)
            z *= _C1
            z ^= z >> np.uint64(27)
            z *= _C2
            z ^= z >> np.uint64(31)
        out[lo:hi] = z.astype(np.uint8)

    with ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 1) as pool:
        list(pool.map(fill, range(0, n, chunk)))
    return out


def _platform():
    from hybridbench.platform import Accounting, Platform

    return Platform.build(1.0, 3.0, accounting=Accounting.MEASURED)


# ------------------------------------------------------------------ legs
# `x`, `keys`, ... : host inputs to reuse (cpu_baseline legs); None → made here


def hist_leg(n: int, x: np.ndarray | None = None, seed: int = 42, bins: int = 256):
    x = splitmix_low8(seed, n) if x is None else x
    if reference_available():
        import_reference()
        from hybridbench.kernels_regular import hybrid_histogram

        p = _platform()
        fn = lambda: hybrid_histogram(x, bins, p)  # noqa: E731
        kind = "reference"
    else:
        from oracle import hist as ohist

        fn = lambda: ohist.hybrid(x, bins, 0.25)  # noqa: E731
        kind = "port"
    m = x.size
    sample = f"2^{m.bit_length() - 1} uint8 through hybrid_histogram, formula share 0.25 (2 side threads)"
    return fn, m, sample, 2, kind, m == n


def sort_leg(n: int, keys: np.ndarray | None = None, seed: int = 42, sample_n: int = 1 << 20):
    m = min(n, sample_n)
    if reference_available():
        import_reference()
        from hybridbench.datasets import gen_sort_data
        from hybridbench.kernels_regular import sample_sort_hybrid

        k = gen_sort_data(m, seed).astype(np.uint32) if keys is None else keys[:m]
        p = _platform()
        fn = lambda: sample_sort_hybrid(k, p)  # noqa: E731
        kind = "reference"
    else:
        from oracle import datasets as ods
        from oracle import sort as osort

        k = (ods.sort_keys(m, seed) if keys is None else keys[:m]).astype(np.int64)
        fn = lambda: osort.sample_sort_hybrid(k, 0.25)  # noqa: E731
        kind = "port"
    return (fn, m, f"2^{m.bit_length() - 1} uint32 keys of gen_sort_data(n, 42), sample_sort_hybrid (keys only)", 2,
            kind, m == n)


def spmv_leg(rows: int, density: float, arrays=None, x: np.ndarray | None = None, seed: int = 42):
    """arrays = (row_ptr, col_idx, values) int64/int64/f64 of gen_csr(rows,
    rows, seed, density) when the caller has them (bit-identical)."""
    if reference_available():
        import_reference()
        from hybridbench.datasets import gen_csr
        from hybridbench.kernels_irregular import CsrMatrix, spmv_hybrid, spmv_preprocess
        from hybridbench.rng import mix_seed, uniform_floats

        m = gen_csr(rows, rows, seed, density) if arrays is None else CsrMatrix(rows, rows, *arrays)
        xx = 2.0 * uniform_floats(mix_seed(seed, 0xDEC0), rows) - 1.0 if x is None else x
        prep = spmv_preprocess(m, _platform())
        nnz = m.nnz
        fn = lambda: spmv_hybrid(prep, xx)  # noqa: E731
        kind = "reference"
    else:
        from oracle import datasets as ods
        from oracle import rng as orng
        from oracle import spmv as ospmv

        ptr, col, val = ods.csr(rows, rows, seed, density) if arrays is None else arrays
        xx = 2.0 * orng.uniform_floats(orng.mix_seed(seed, 0xDEC0), rows) - 1.0 if x is None else x
        perm, permuted, split = ospmv.preprocess(ptr, col, val, 1.0, 3.0, None)
        nnz = int(ptr[-1])
        fn = lambda: ospmv.hybrid(perm, permuted, split, xx)  # noqa: E731
        kind = "port"
    return (fn, 2 * nnz, f"gen_csr({rows}, {rows}, 42, {density}), spmv_hybrid (prep untimed), modeled split", 2,
            kind, True)


def filter_leg(kind_name: str, side: int, radius: int, img: np.ndarray | None = None, rows: int = 64,
               seed: int = 42):
    if img is None:
        img = splitmix_low8(seed, (rows + radius) * side).reshape(rows + radius, side)
    img = np.ascontiguousarray(img[:rows])
    if reference_available():
        import_reference()
        from hybridbench.kernels_regular import FilterKernel, Image, build_bilateral_lut, hybrid_bilateral, hybrid_convolve

        p = _platform()
        if kind_name == "bilat":
            lut = build_bilateral_lut(radius, max(radius / 2.0, 0.5), 40.0)
            fn = lambda: hybrid_bilateral(Image(img), lut, p)  # noqa: E731
        else:
            fk = FilterKernel.gaussian(radius)
            fn = lambda: hybrid_convolve(Image(img), fk, p)  # noqa: E731
        kind = "reference"
    else:
        from oracle import bilateral as obil
        from oracle import conv as oconv

        if kind_name == "bilat":
            sp, rg = obil.lut(radius, max(radius / 2.0, 0.5), 40.0)
            fn = lambda: obil.hybrid(img, sp, rg, radius, 0.25)  # noqa: E731
        else:
            ax = np.arange(-radius, radius + 1, dtype=np.float64)
            sg = max(radius / 2.0, 0.5)
            g = np.exp(-(ax[:, None] ** 2 + ax[None, :] ** 2) / (2.0 * sg**2))
            w = g / g.sum()
            fn = lambda: oconv.hybrid(img, w, 0.25)  # noqa: E731
        kind = "port"
    what = "hybrid_bilateral" if kind_name == "bilat" else "hybrid_convolve"
    return fn, rows * side, f"{rows} x {side} strip of gen_image({side}, 42), {what}", 2, kind, False


def lr_leg(n: int, seed: int = 42, sample_n: int = 1 << 20):
    m = min(n, sample_n)
    if reference_available():
        import_reference()
        from hybridbench.datasets import gen_list
        from hybridbench.kernels_irregular import list_rank_with_stats

        lst = gen_list(m, seed)
        p = _platform()
        fn = lambda: list_rank_with_stats(lst, p, seed)  # noqa: E731
        kind = "reference"
    else:
        from oracle import datasets as ods
        from oracle import listrank as olr

        succ, head = ods.linked_list(m, seed)
        fn = lambda: olr.list_rank_with_stats(succ, head, seed)  # noqa: E731
        kind = "port"
    return fn, m, f"gen_list(2^{m.bit_length() - 1}, 42), list_rank_with_stats", 1, kind, m == n
