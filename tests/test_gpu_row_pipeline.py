"""Host-buffer filter calls large enough for the chunked H2D / kernel / D2H
pipeline (runtime.cu row_pipeline, > 128 MB of output): bit-identical to the
device-resident call (itself pinned to the oracle and the reference's golden
outputs elsewhere) and, on sampled strips, to the oracle — whole images,
ranges that do not line up with the chunk grid, f64 and u8 input, f32 and
f64 output, pageable and pinned results."""

import numpy as np
import pytest
import torch

from oracle import bilateral as obil
from oracle import conv as oconv
from oracle import datasets as ods
from paper_1303_2171_b200.kernels_regular import (
    FilterKernel,
    build_bilateral_lut,
    gpu_bilateral_rows,
    gpu_convolve_rows,
)

pytestmark = pytest.mark.gpu
H, W = 4400, 4100  # 144 MB of f64 output: 4 chunks of 32 MB; f32: 2


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a.view(np.uint32)


@pytest.fixture(scope="module")
def img():
    return np.ascontiguousarray(ods.image(H, 11)[:, :W])


@pytest.mark.parametrize("out_dtype", [np.float64, np.float32])
@pytest.mark.parametrize("rows", [(0, H), (3, H - 5), (1111, 4321)])
def test_convolution_host_pipeline(img, rows, out_dtype):
    k = FilterKernel.gaussian(3)
    r0, r1 = rows
    dev = gpu_convolve_rows(torch.from_numpy(img).cuda(), k, r0, r1, out_dtype=out_dtype).cpu().numpy()
    host = gpu_convolve_rows(img, k, r0, r1, out_dtype=out_dtype)
    assert np.array_equal(bits(host), bits(dev))
    for a in (r0, (r0 + r1) // 2, r1 - 4):
        want = oconv.rows(img, k.weights, a, a + 4).astype(out_dtype)
        assert np.array_equal(bits(host[a - r0 : a - r0 + 4]), bits(want))
    # f64 input, into a caller-provided pageable result
    f = img.astype(np.float64) * 0.5
    out = np.empty((r1 - r0, W), dtype=out_dtype)
    gpu_convolve_rows(f, k, r0, r1, out=out, out_dtype=out_dtype)
    want = oconv.rows(f, k.weights, r1 - 3, r1).astype(out_dtype)
    assert np.array_equal(bits(out[-3:]), bits(want))


@pytest.mark.parametrize("rows", [(0, H), (2049, 4397)])
def test_bilateral_host_pipeline(img, rows):
    lut = build_bilateral_lut(4, 2.0, 30.0)
    r0, r1 = rows
    dev = gpu_bilateral_rows(torch.from_numpy(img).cuda(), lut, r0, r1).cpu().numpy()
    host = gpu_bilateral_rows(img, lut, r0, r1)
    assert np.array_equal(bits(host), bits(dev))
    sp, rg = lut.spatial_weights, lut.range_weights
    for a in (r0, r1 - 2):
        want = obil.rows(img, sp, rg, 4, a, a + 2)
        assert np.array_equal(bits(host[a - r0 : a - r0 + 2]), bits(want))


def test_host_empty_pins_only_when_it_pays_back(monkeypatch):
    """host_empty never makes the library pin fresh memory for a caller that
    keeps its results: a first result is pageable; once the caller drops a
    result of a size class (and holds none), the next one is page-locked
    once and its block is reused by every later call; results of one API
    call (result_scope) do not hold each other back."""
    import gc

    import torch

    from paper_1303_2171_b200 import gpu
    from paper_1303_2171_b200.gpu import host_empty, result_scope

    def pinned(a):
        return torch.from_numpy(a).is_pinned()

    gc.collect()
    monkeypatch.setattr(gpu, "_pool", gpu._ResultPool())  # no history from earlier tests
    n = (1 << 21) + 1000  # 2^25-byte size class
    a = host_empty(n)
    assert not pinned(a) and a.shape == (n,) and a.dtype == np.float64  # first result: pageable
    b = host_empty(n)
    assert not pinned(b)  # `a` held, nothing dropped yet
    del a, b
    gc.collect()
    c = host_empty(n)  # the caller drops its results: pin once
    assert pinned(c)
    d = host_empty(n)  # `c` held: pageable (no fresh pin per call)
    assert not pinned(d)
    del c, d
    gc.collect()
    e = host_empty(n)  # c's block, reused
    assert pinned(e)
    del e
    gc.collect()
    with result_scope():
        k, v = host_empty(n), host_empty(n)
    assert pinned(k) and pinned(v)
    del k, v
    gc.collect()
    # gpu_sort: keys + payload of one call, dropped between calls
    from paper_1303_2171_b200.kernels_regular import gpu_sort

    keys = np.random.default_rng(3).integers(0, 1 << 32, size=(1 << 23) + 5, dtype=np.uint32)
    first = gpu_sort(keys, np.arange(keys.size, dtype=np.uint32))
    assert np.array_equal(first[0], np.sort(keys)) and np.array_equal(keys[first[1]], first[0])
    del first
    gc.collect()
    for _ in range(2):
        sk, sv, _ = gpu_sort(keys, np.arange(keys.size, dtype=np.uint32))
        assert pinned(sk) and pinned(sv)
        assert np.array_equal(sk, np.sort(keys)) and np.array_equal(keys[sv], sk)
        del sk, sv
        gc.collect()
