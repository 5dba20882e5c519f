"""The reference's acceptance criteria that cover the hot path, run through
this package's drop-in API with the GPU share on the B200 (reference
tests/test_acceptance.py): criterion 3 (split invariance over the 11-point
share grid, 20 instances per kernel, against independent oracles) and the
list-ranking half of criterion 5 (50 lists, ranks = pointer chasing, FIS
reduced size <= n / log2 n).  Criterion 7 (the 3600^2 convolution figure)
is tests/test_gpu_conv.py::test_criterion_7_figure_reproduction.  On top of
the reference's tolerances, every result must be bit-identical to the share-0
(all-GPU) result: split invariance is exact here."""

import math

import numpy as np
import pytest

from oracle import bilateral as obil
from oracle import hist as ohist
from oracle import listrank as olr
from paper_1303_2171_b200.datasets import gen_csr, gen_hist_data, gen_image, gen_list, gen_sort_data
from paper_1303_2171_b200.kernels_irregular import list_rank_with_stats, spmv_hybrid, spmv_preprocess
from paper_1303_2171_b200.kernels_regular import (
    FilterKernel,
    build_bilateral_lut,
    hybrid_bilateral,
    hybrid_convolve,
    hybrid_histogram,
    hybrid_sort,
)
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.rng import mix_seed, uniform_floats
from paper_1303_2171_b200.worksharing import WorkShare

pytestmark = pytest.mark.gpu
SHARES = [i / 10 for i in range(11)]


def _naive_convolve(px, w):
    """Direct clamp-to-edge correlation, one pixel at a time (independent of
    the row-plane order of the reference and of the kernels)."""
    h, wd = px.shape
    r = w.shape[0] // 2
    out = np.zeros((h, wd))
    for y in range(h):
        for x in range(wd):
            acc = 0.0
            for dy in range(-r, r + 1):
                for dx in range(-r, r + 1):
                    acc += w[dy + r, dx + r] * float(px[min(max(y + dy, 0), h - 1), min(max(x + dx, 0), wd - 1)])
            out[y, x] = acc
    return out


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def test_criterion_3_split_invariance():
    p = Platform.build(1.0, 3.0)
    checked = 0
    for seed in range(20):
        data = gen_hist_data(1_500, seed=seed, bins=64)
        want = ohist.sequential(data, 64)
        for share in SHARES:
            assert np.array_equal(hybrid_histogram(data, 64, p, WorkShare.manual(share)).bins, want)
        checked += 1
    for seed in range(20, 40):
        data = gen_sort_data(1_200, seed=seed)
        want = np.sort(data)
        for share in SHARES:
            assert np.array_equal(hybrid_sort(data, p, share=WorkShare.manual(share)), want)
        checked += 1
    for seed in range(40, 60):
        img = gen_image(20, seed=seed)
        w = uniform_floats(mix_seed(seed, 1), 25).reshape(5, 5) * 2 - 1
        want = _naive_convolve(img.pixels, w)
        base = None
        for share in SHARES:
            got = np.asarray(hybrid_convolve(img, FilterKernel(w), p, WorkShare.manual(share)).pixels)
            assert np.allclose(got, want, rtol=1e-6, atol=1e-9)
            base = got if base is None else base
            assert np.array_equal(_bits(got), _bits(base))
        checked += 1
    for seed in range(60, 80):
        img = gen_image(14, seed=seed)
        lut = build_bilateral_lut(2, 1.8, 28.0)
        want = obil.direct(img.pixels, 2, 1.8, 28.0)
        base = None
        for share in SHARES:
            got = np.asarray(hybrid_bilateral(img, lut, p, WorkShare.manual(share)).pixels)
            assert np.allclose(got, want, rtol=1e-5, atol=1e-8)
            base = got if base is None else base
            assert np.array_equal(_bits(got), _bits(base))
        checked += 1
    for seed in range(80, 100):
        m = gen_csr(36, 36, seed=seed, density=0.12)
        x = uniform_floats(mix_seed(seed, 2), 36) * 2 - 1
        dense = np.zeros((36, 36))
        rows = np.repeat(np.arange(36), np.diff(np.asarray(m.row_ptr)))
        dense[rows, np.asarray(m.col_idx)] = np.asarray(m.values)
        want = dense @ x
        base = None
        for share in SHARES:
            got = np.asarray(spmv_hybrid(spmv_preprocess(m, p, WorkShare.manual(share)), x))
            assert np.allclose(got, want, rtol=1e-6, atol=1e-12)
            base = got if base is None else base
            assert np.array_equal(_bits(got), _bits(base))
        checked += 1
    assert checked == 100


def test_criterion_5_list_ranking():
    p = Platform.build(1.0, 3.0)
    for i in range(50):
        n = 100 + (mix_seed(i, 5) % 9_901)
        lst = gen_list(int(n), seed=i)
        ranks, stats = list_rank_with_stats(lst, p, seed=i)
        assert np.array_equal(np.asarray(ranks), olr.chase(np.asarray(lst.succ), lst.head)), i
        assert stats.reduced_size <= n / math.log2(n), i
