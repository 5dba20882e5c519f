"""Bilateral GPU parity: bit-identical (fp64) to the reference's own outputs
and to the oracle strips, for every share; mirrors the reference's
tests/test_kernels_regular.py:184-234 and acceptance :144-151."""

import numpy as np
import pytest

from conftest import golden
from oracle import bilateral as obil
from oracle import datasets as ods
from paper_1303_2171_b200.kernels_regular import (
    BilateralApplyWorkload,
    Image,
    build_bilateral_lut,
    gpu_bilateral_rows,
    hybrid_bilateral,
)
from paper_1303_2171_b200.worksharing import WorkShare

pytestmark = pytest.mark.gpu
SHARES = [i / 10 for i in range(11)]


def test_golden_bit_exact(platform13):
    g = golden("bilateral")
    for i in range(4):
        side, seed, radius, ss, sr = g[f"meta_{i}"]
        radius = int(radius)
        img = Image(g[f"img_{i}"])
        lut = build_bilateral_lut(radius, float(ss), float(sr))
        assert np.array_equal(lut.spatial_weights, g[f"spatial_{i}"])
        out = hybrid_bilateral(img, lut, platform13)
        assert np.array_equal(out.pixels, g[f"out_{i}"])
        s3 = int(side) // 3
        assert np.array_equal(gpu_bilateral_rows(img.pixels, lut, s3, s3 + 5), g[f"strip_{i}"])
    lut = build_bilateral_lut(3, 2.0, 25.0)
    assert np.array_equal(hybrid_bilateral(Image(g["rect_img"]), lut, platform13).pixels, g["rect_out"])


def test_split_invariance_bit_exact(platform13):
    img = Image(ods.image(30, 6))
    lut = build_bilateral_lut(2, 1.5, 20.0)
    ref = hybrid_bilateral(img, lut, platform13, WorkShare.manual(0.5)).pixels
    for share in SHARES:
        assert np.array_equal(hybrid_bilateral(img, lut, platform13, WorkShare.manual(share)).pixels, ref)


def test_share_one_equals_device_a(platform13):
    img = Image(ods.image(24, 8))
    lut = build_bilateral_lut(2, 2.0, 30.0)
    solo = BilateralApplyWorkload(img, lut).run_part(platform13.device_a, (0, img.height))
    assert np.array_equal(hybrid_bilateral(img, lut, platform13, WorkShare.manual(0.0)).pixels, solo)


@pytest.mark.parametrize("radius", [0, 1, 3, 5, 7, 8, 9])
def test_radii_and_ragged_shapes(radius):
    pix = ods.image(97, 11)[:, :83].copy()  # width not a multiple of the tile
    sp, rg = obil.lut(radius, max(radius / 2.0, 0.5), 40.0)
    lut = build_bilateral_lut(radius, max(radius / 2.0, 0.5), 40.0)
    for r0, r1 in ((0, 97), (5, 6), (40, 77), (90, 97)):
        want = obil.rows(pix, sp, rg, radius, r0, r1)
        assert np.array_equal(gpu_bilateral_rows(pix, lut, r0, r1), want)


def test_flat_image_fixed_point(platform13):
    for radius in (1, 3, 5):
        lut = build_bilateral_lut(radius, 2.0, 25.0)
        out = hybrid_bilateral(Image(np.full((20, 20), 137, dtype=np.uint8)), lut, platform13)
        assert np.allclose(out.pixels, 137.0, rtol=0, atol=1e-9)


def test_lut_free_oracle_and_fp32_tolerance():
    pix = ods.image(64, 4)
    lut = build_bilateral_lut(3, 2.5, 35.0)
    want = obil.direct(pix, 3, 2.5, 35.0)
    assert np.allclose(gpu_bilateral_rows(pix, lut, 0, 64), want, rtol=1e-5, atol=1e-8)
    f32 = gpu_bilateral_rows(pix, lut, 0, 64, out_dtype=np.float32)
    assert f32.dtype == np.float32
    assert np.allclose(f32, want, rtol=1e-5, atol=1e-8)


def test_device_resident_path():
    import torch

    pix = ods.image(300, 42)
    lut = build_bilateral_lut(5, 2.5, 40.0)
    sp, rg = obil.lut(5, 2.5, 40.0)
    d = torch.from_numpy(pix).cuda()
    got = gpu_bilateral_rows(d, lut, 17, 250).cpu().numpy()
    assert np.array_equal(got, obil.rows(pix, sp, rg, 5, 17, 250))


@pytest.mark.parametrize("radius", [0, 2, 5, 8])
def test_tma_staged_tiles_bit_exact(radius):
    # widths that are multiples of 16 take the TMA-staged kernel (interior
    # tiles by one 2-D tensor copy, border tiles by clamped loads)
    import torch

    pix = ods.image(400, 21)[:, :368].copy()  # 368 % 16 == 0, not a multiple of the 64-wide tile
    lut = build_bilateral_lut(radius, max(radius / 2.0, 0.5), 30.0)
    sp, rg = obil.lut(radius, max(radius / 2.0, 0.5), 30.0)
    d = torch.from_numpy(pix).cuda()
    for r0, r1 in ((0, 400), (37, 301), (399, 400)):
        got = gpu_bilateral_rows(d, lut, r0, r1).cpu().numpy()
        assert np.array_equal(got, obil.rows(pix, sp, rg, radius, r0, r1)), (radius, r0, r1)


@pytest.mark.parametrize("radius", [0, 1, 5, 7])
def test_fp32_arithmetic_within_tolerance(radius):
    """arithmetic="fp32" (fp32 taps, FMA): within 1e-5 relative of the fp64
    reference arithmetic (north_star's filter tolerance), host and device
    paths, fp32 and fp64 outputs, through the public API too."""
    import torch

    from oracle import bilateral as obil
    from oracle import datasets as ods
    from paper_1303_2171_b200.kernels_regular import Image, build_bilateral_lut, gpu_bilateral_rows, hybrid_bilateral
    from paper_1303_2171_b200.platform import Platform

    img = ods.image(301, radius + 3)
    sig = max(radius / 2.0, 0.5)
    lut = build_bilateral_lut(radius, sig, 40.0)
    sp, rg = obil.lut(radius, sig, 40.0)
    want = obil.rows(img, sp, rg, radius, 0, 301)
    for out_dtype in (np.float32, np.float64):
        got = gpu_bilateral_rows(torch.from_numpy(img).cuda(), lut, 0, 301, out_dtype=out_dtype, arithmetic="fp32")
        assert np.allclose(got.cpu().numpy(), want, rtol=1e-5, atol=0), out_dtype
        host = gpu_bilateral_rows(img, lut, 10, 200, out_dtype=out_dtype, arithmetic="fp32")
        assert np.allclose(host, want[10:200], rtol=1e-5, atol=0)
    res = hybrid_bilateral(Image(img), lut, Platform.build(1.0, 3.0), arithmetic="fp32").pixels
    assert np.allclose(res, want, rtol=1e-5, atol=0)
    with pytest.raises(ValueError):
        gpu_bilateral_rows(img, lut, 0, 4, arithmetic="fp16")
