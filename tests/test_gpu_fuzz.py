"""Randomised parity of the public drop-in API (hypothesis): random sizes,
dtypes, shares, host vs device inputs, every result compared with the oracle
restatement of the reference (bit-exact for integer work and for the fp64
SpMV / filters).  Complements the fixed-case tests with shapes nobody chose:
ragged sizes, tiny and empty inputs, shares at and near 0 and 1."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import bilateral as obil
from oracle import conv as oconv
from oracle import datasets as ods
from oracle import hist as ohist
from oracle import listrank as olr
from oracle import sort as osort
from oracle import spmv as ospmv

pytestmark = pytest.mark.gpu
FUZZ = settings(max_examples=150, deadline=None, derandomize=True,
                suppress_health_check=[HealthCheck.too_slow, HealthCheck.data_too_large])
SHARES = st.one_of(st.sampled_from([0.0, 1.0, 0.25, 0.5]), st.floats(0.0, 1.0))


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def _share(f):
    from paper_1303_2171_b200.worksharing import WorkShare

    return WorkShare.manual(f)


def _platform():
    from paper_1303_2171_b200.platform import Platform

    return Platform.build(1.0, 3.0)


@FUZZ
@given(n=st.integers(0, 70_000), bins=st.sampled_from([1, 2, 7, 255, 256, 1000]),
       dtype=st.sampled_from(["u1", "i2", "u4", "i8"]), share=SHARES, device=st.booleans(),
       seed=st.integers(0, 2**31))
def test_histogram(n, bins, dtype, share, device, seed):
    import torch

    from paper_1303_2171_b200.kernels_regular import hybrid_histogram

    if dtype == "u1" and bins > 256:
        bins = 256
    data = (np.random.default_rng(seed).integers(0, bins, size=n)).astype(np.dtype(dtype))
    want = ohist.sequential(data, bins)
    arg = torch.from_numpy(data).cuda() if device and n else data
    if n == 0:  # the reference's engine: an empty modeled timeline is a ValueError
        with pytest.raises(ValueError, match="timeline is empty"):
            hybrid_histogram(arg, bins, _platform(), _share(share))
        return
    got = np.asarray(hybrid_histogram(arg, bins, _platform(), _share(share)).bins)
    assert np.array_equal(got, want)


@FUZZ
@given(n=st.integers(0, 60_000), dtype=st.sampled_from(["u4", "i4", "u8", "i8", "u2"]), share=SHARES,
       span=st.sampled_from([1, 3, 1000, 2**31]), seed=st.integers(0, 2**31))
def test_sort(n, dtype, share, span, seed):
    from paper_1303_2171_b200.kernels_regular import sample_sort_hybrid

    dt = np.dtype(dtype)
    info = np.iinfo(dt)
    lo = max(info.min, -span) if info.min < 0 else 0
    hi = min(info.max, lo + span)
    data = np.random.default_rng(seed).integers(lo, hi, size=n, endpoint=True).astype(dt)
    out, wa, wb = sample_sort_hybrid(data, _platform(), share=_share(share))
    ref_out, ref_a, ref_b = osort.sample_sort_hybrid(data, share)
    assert np.asarray(out).dtype == dt
    assert np.array_equal(np.asarray(out), ref_out) and (wa, wb) == (ref_a, ref_b)


@FUZZ
@given(rows=st.integers(1, 3_000), cols=st.integers(1, 3_000), dens=st.floats(1e-4, 0.02), share=SHARES,
       device=st.booleans(), seed=st.integers(0, 2**31))
def test_spmv(rows, cols, dens, share, device, seed):
    import torch

    from oracle import rng as orng
    from paper_1303_2171_b200.kernels_irregular import CsrMatrix, spmv_hybrid, spmv_preprocess

    ptr, col, val = ods.csr(rows, cols, seed % 10_000, dens)
    x = 2.0 * orng.uniform_floats(orng.mix_seed(seed % 10_000, 0xDEC0), cols) - 1.0
    m = CsrMatrix(rows, cols, ptr, col, val)
    if device:
        m = m.to_device()
    prep = spmv_preprocess(m, _platform(), _share(share))
    y = spmv_hybrid(prep, torch.from_numpy(x).cuda() if device else x)
    y = y.cpu().numpy() if hasattr(y, "cpu") else np.asarray(y)
    perm, permuted, split = ospmv.preprocess(ptr, col, val, 1.0, 3.0, share)
    assert int(prep.split_row) == int(split)
    assert np.array_equal(_bits(y), _bits(ospmv.hybrid(perm, permuted, split, x)))


@FUZZ
@given(h=st.integers(1, 90), w=st.integers(1, 90), r=st.integers(0, 6), share=SHARES,
       device=st.booleans(), seed=st.integers(0, 2**31))
def test_filters(h, w, r, share, device, seed):
    import torch

    from paper_1303_2171_b200.kernels_regular import (
        FilterKernel,
        Image,
        build_bilateral_lut,
        hybrid_bilateral,
        hybrid_convolve,
    )

    rng = np.random.default_rng(seed)
    px = rng.integers(0, 256, size=(h, w), dtype=np.uint8)
    wts = rng.uniform(-1, 1, size=(2 * r + 1, 2 * r + 1))
    wts[rng.random(wts.shape) < 0.2] = 0.0  # zero taps are skipped, like the reference
    img = Image(torch.from_numpy(px).cuda() if device else px)
    got = hybrid_convolve(img, FilterKernel(wts), _platform(), _share(share)).pixels
    got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
    assert np.array_equal(_bits(got), _bits(oconv.hybrid(px, wts, share)))
    sigma_s, sigma_r = max(r / 2, 0.5), 40.0
    lut = build_bilateral_lut(r, sigma_s, sigma_r)
    got = hybrid_bilateral(img, lut, _platform(), _share(share)).pixels
    got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
    sp, rg = obil.lut(r, sigma_s, sigma_r)
    assert np.array_equal(_bits(got), _bits(obil.hybrid(px, sp, rg, r, share)))


@FUZZ
@given(n=st.integers(1, 40_000), seed=st.integers(0, 2**31), device=st.booleans(),
       wide=st.booleans())
def test_list_rank(n, seed, device, wide):
    import torch

    from paper_1303_2171_b200.kernels_irregular import LinkedListArr, list_rank_hybrid

    succ, head = ods.linked_list(n, seed % 100_000)
    succ = succ.astype(np.int64 if wide else np.int32)
    arg = torch.from_numpy(succ).cuda() if device else succ
    got = list_rank_hybrid(LinkedListArr(arg, head), _platform(), seed % 1000)
    got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
    assert np.array_equal(got, olr.chase(succ.astype(np.int64), head))
