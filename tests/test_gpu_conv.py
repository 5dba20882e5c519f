"""Convolution GPU parity: bit-identical (fp64) to the reference's own
outputs (tests/golden/conv.npz) and to the oracle strips, for every share;
mirrors the reference's tests/test_kernels_regular.py:123-175 and
acceptance criterion 7 (tests/test_acceptance.py:255-276)."""

import numpy as np
import pytest

from conftest import golden
from oracle import conv as oconv
from oracle import datasets as ods
from oracle import rng as orng
from paper_1303_2171_b200.kernels_regular import (
    ConvolutionWorkload,
    FilterKernel,
    Image,
    gpu_convolve_rows,
    hybrid_convolve,
)
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

pytestmark = pytest.mark.gpu
SHARES = [i / 10 for i in range(11)]


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def test_golden_bit_exact(platform13):
    g = golden("conv")
    for i in range(6):
        img, k = Image(g[f"img_{i}"]), FilterKernel(g[f"w_{i}"])
        for j, share in enumerate((0.0, 0.3, 1.0)):
            out = hybrid_convolve(img, k, platform13, WorkShare.manual(share)).pixels
            assert np.array_equal(bits(out), bits(g[f"out_{i}"][j])), (i, share)
        s3 = img.height // 3
        assert np.array_equal(bits(gpu_convolve_rows(img.pixels, k, s3, s3 + 5)), bits(g[f"strip_{i}"]))
    out = hybrid_convolve(Image(g["f64_img"]), FilterKernel(g["f64_w"]), platform13, WorkShare.manual(0.0))
    assert np.array_equal(bits(out.pixels), bits(g["f64_out"]))
    out = hybrid_convolve(Image(g["rect_img"]), FilterKernel(g["f64_w"]), platform13, WorkShare.manual(0.0))
    assert np.array_equal(bits(out.pixels), bits(g["rect_out"]))


def test_delta_kernel_is_identity(platform13):
    img = Image(ods.image(32, 5))
    out = hybrid_convolve(img, FilterKernel.delta(2), platform13, WorkShare.manual(0.0))
    assert np.array_equal(out.pixels, img.pixels.astype(np.float64))


def test_strip_sizes_for_18_percent():
    wl = ConvolutionWorkload(Image(np.zeros((3600, 3600), dtype=np.uint8)), FilterKernel.delta(7))
    assert wl.partition(0.18) == ((0, 648), (648, 3600))


def test_matches_naive_within_reference_tolerance(platform13):
    img = ods.image(24, 9)
    w = orng.uniform_floats(123, 25).reshape(5, 5) * 2 - 1
    h, wd = img.shape
    naive = np.zeros((h, wd))
    for y in range(h):
        for x in range(wd):
            acc = 0.0
            for dy in range(-2, 3):
                for dx in range(-2, 3):
                    acc += w[dy + 2, dx + 2] * float(img[min(max(y + dy, 0), h - 1), min(max(x + dx, 0), wd - 1)])
            naive[y, x] = acc
    out = hybrid_convolve(Image(img), FilterKernel(w), platform13, WorkShare.manual(0.0))
    assert np.allclose(out.pixels, naive, rtol=1e-6, atol=1e-9)


def test_split_invariance_bit_exact(platform13):
    img = Image(ods.image(40, 3))
    k = FilterKernel.gaussian(3)
    ref = hybrid_convolve(img, k, platform13, WorkShare.manual(0.0)).pixels
    for share in SHARES:
        assert np.array_equal(hybrid_convolve(img, k, platform13, WorkShare.manual(share)).pixels, ref)


def test_linearity(platform13):
    k = FilterKernel.gaussian(2)
    a = ods.image(16, 1).astype(np.float64)
    b = ods.image(16, 2).astype(np.float64)
    s = WorkShare.manual(0.0)
    combo = hybrid_convolve(Image(0.7 * a - 1.3 * b), k, platform13, s).pixels
    sep = 0.7 * hybrid_convolve(Image(a), k, platform13, s).pixels - 1.3 * hybrid_convolve(Image(b), k, platform13, s).pixels
    assert np.allclose(combo, sep, rtol=1e-6, atol=1e-9)


@pytest.mark.parametrize("radius", [0, 1, 4, 7, 8, 9, 12])
def test_radii_ragged_shapes_and_zero_taps(radius):
    pix = ods.image(97, 11)[:, :83].copy()
    side = 2 * radius + 1
    w = orng.uniform_floats(radius + 5, side * side).reshape(side, side) - 0.5
    w[::2, 1::3] = 0.0  # zero taps are skipped, as in the reference
    for r0, r1 in ((0, 97), (5, 6), (40, 77), (90, 97)):
        want = oconv.rows(pix, w, r0, r1)
        assert np.array_equal(bits(gpu_convolve_rows(pix, FilterKernel(w), r0, r1)), bits(want)), (radius, r0)


def test_input_dtypes_and_fp32_output():
    pix = ods.image(50, 8)
    k = FilterKernel.gaussian(3)
    want = oconv.rows(pix, k.weights, 0, 50)
    for dt in (np.uint8, np.int32, np.float32, np.float64, np.uint16):
        assert np.array_equal(bits(gpu_convolve_rows(pix.astype(dt), k, 0, 50)), bits(want)), dt
    f32 = gpu_convolve_rows(pix, k, 0, 50, out_dtype=np.float32)
    assert f32.dtype == np.float32 and np.array_equal(f32, want.astype(np.float32))


def test_device_resident_path():
    import torch

    pix = ods.image(300, 42)
    k = FilterKernel.gaussian(7)
    want = oconv.rows(pix, k.weights, 17, 250)
    for t in (torch.from_numpy(pix).cuda(), torch.from_numpy(pix.astype(np.float64)).cuda(),
              torch.from_numpy(pix.astype(np.int16)).cuda()):
        got = gpu_convolve_rows(t, k, 17, 250).cpu().numpy()
        assert np.array_equal(bits(got), bits(want))


def test_criterion_7_figure_reproduction():
    import scipy.ndimage

    from paper_1303_2171_b200.platform import modeled_compute_time
    from paper_1303_2171_b200.worksharing import calibrate

    platform = Platform.build(18.0, 82.0)
    share = calibrate(platform, lambda d, w: modeled_compute_time(d, w), sample=3600.0 * 3600.0, max_refinements=8)
    assert share.fraction_a == pytest.approx(0.18, abs=1e-12)
    img = Image(ods.image(3600, 42))
    k = FilterKernel.gaussian(7)
    assert ConvolutionWorkload(img, k).partition(share.fraction_a) == ((0, 648), (648, 3600))
    out = hybrid_convolve(img, k, platform, share)
    expected = scipy.ndimage.correlate(img.pixels.astype(np.float64), k.weights, mode="nearest")
    assert np.allclose(out.pixels, expected, rtol=1e-6, atol=1e-9)
    # and bit-exact with the reference arithmetic on a strip from each side
    for r0 in (600, 2000):
        assert np.array_equal(bits(out.pixels[r0 : r0 + 64]), bits(oconv.rows(img.pixels, k.weights, r0, r0 + 64)))


@pytest.mark.parametrize("radius", [0, 2, 7, 8])
def test_fp32_arithmetic_within_tolerance(radius):
    """arithmetic="fp32": fp32 taps with FMA, within 1e-5 relative of the fp64
    reference arithmetic (absolute floor: 1e-5 of the largest possible
    |output|, for outputs near zero with signed weights); uint8 and float64
    images, zero taps, the public API."""
    import torch

    from oracle import conv as oconv
    from oracle import datasets as ods
    from paper_1303_2171_b200.kernels_regular import FilterKernel, Image, gpu_convolve_rows, hybrid_convolve
    from paper_1303_2171_b200.platform import Platform

    rs = np.random.default_rng(radius)
    img = ods.image(211, radius + 5)
    for fk in (FilterKernel.gaussian(radius), FilterKernel(rs.standard_normal((2 * radius + 1,) * 2))):
        w = fk.weights.copy()
        if w.size > 1:
            w.flat[::3] = 0.0  # zero taps
        fk = FilterKernel(w)
        for pix in (img, img.astype(np.float64) / 7.0):
            want = oconv.rows(pix, fk.weights, 0, 211)
            scale = np.abs(fk.weights).sum() * np.abs(pix).max()
            got = gpu_convolve_rows(torch.from_numpy(pix).cuda(), fk, 0, 211, out_dtype=np.float32, arithmetic="fp32")
            assert np.allclose(got.cpu().numpy(), want, rtol=1e-5, atol=1e-5 * scale)
            host = gpu_convolve_rows(pix, fk, 3, 150, arithmetic="fp32")
            assert np.allclose(host, want[3:150], rtol=1e-5, atol=1e-5 * scale)
    res = hybrid_convolve(Image(img), FilterKernel.gaussian(radius), Platform.build(1.0, 3.0), arithmetic="fp32").pixels
    assert np.allclose(res, oconv.rows(img, FilterKernel.gaussian(radius).weights, 0, 211), rtol=1e-5, atol=1e-5 * 255)
