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
