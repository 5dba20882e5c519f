"""Native DeviceA (host-core) kernels: bit-identical to
the reference's numpy bodies / golden outputs, on any worker count.  CPU only
— libhb200.so loads and runs these without a GPU."""

import numpy as np
import pytest

from conftest import golden
from oracle import bilateral as obil
from oracle import conv as oconv
from oracle import datasets as ods
from paper_1303_2171_b200.kernels_irregular import CsrMatrix, _host_range_matvec
from paper_1303_2171_b200.kernels_regular import (
    FilterKernel,
    HistogramWorkload,
    bilateral_rows,
    build_bilateral_lut,
    convolve_rows,
    host_histogram,
)
from paper_1303_2171_b200.platform import Platform


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("workers", [1, 3, 8])
def test_host_histogram_golden(workers):
    g = golden("hist")
    for i in range(4):
        n, seed, bins = g[f"meta_{i}"]
        data = g[f"data_{i}"]
        want = g[f"bins_{i}"][0]
        for dt in (np.uint8, np.int16, np.uint32, np.int64, np.uint64):
            if bins > 256 and dt == np.uint8:
                continue
            assert np.array_equal(host_histogram(data.astype(dt), int(bins), workers), want), (i, dt)


def test_host_histogram_errors():
    with pytest.raises(ValueError):
        host_histogram(np.array([0, 5, 300], dtype=np.int64), 256, 2)
    with pytest.raises(ValueError):
        host_histogram(np.array([-1], dtype=np.int8), 4, 1)
    with pytest.raises(TypeError):
        host_histogram(np.array([1.0]), 4, 1)
    assert host_histogram(np.zeros(0, dtype=np.uint8), 7, 4).sum() == 0


def test_device_a_side_of_workload_is_native_and_exact():
    data = ods.hist_values(100_001, 3, 256).astype(np.uint8)
    p = Platform.build(1.0, 3.0)
    wl = HistogramWorkload(data, 256)
    a, _ = wl.partition(1.0)
    assert np.array_equal(wl.run_part(p.device_a, a), np.bincount(data, minlength=256))


@pytest.mark.parametrize("workers", [1, 4])
def test_host_spmv_rows_golden(workers):
    g = golden("spmv")
    for i in range(4):
        ptr, col, val, x = g[f"ptr_{i}"], g[f"col_{i}"], g[f"val_{i}"], g[f"x_{i}"]
        m = CsrMatrix(ptr.size - 1, x.size, ptr, col, val)
        from oracle import spmv as ospmv

        want = ospmv.sequential_rows(ptr, col, val, x) if ptr.size < 3000 else ospmv.range_matvec(ptr, col, val, x, 0, ptr.size - 1)
        got = _host_range_matvec(m, x, 0, m.rows, workers)
        assert np.array_equal(bits(got), bits(want)), i
        r0, r1 = m.rows // 3, m.rows // 2
        assert np.array_equal(bits(_host_range_matvec(m, x, r0, r1, workers)), bits(want[r0:r1]))
    m32 = CsrMatrix(ptr.size - 1, x.size, ptr.astype(np.int32), col.astype(np.int32), val)
    assert np.array_equal(bits(_host_range_matvec(m32, x, 0, m32.rows, 2)), bits(want))


@pytest.mark.parametrize("workers", [1, 5])
def test_host_conv_rows_golden(workers):
    g = golden("conv")
    for i in range(6):
        img, w = g[f"img_{i}"], g[f"w_{i}"]
        k = FilterKernel(w)
        assert np.array_equal(bits(convolve_rows(img, k, 0, img.shape[0], workers)), bits(g[f"out_{i}"][0])), i
        s3 = img.shape[0] // 3
        assert np.array_equal(bits(convolve_rows(img, k, s3, s3 + 5, workers)), bits(g[f"strip_{i}"]))
    got = convolve_rows(g["f64_img"], FilterKernel(g["f64_w"]), 0, 16, workers)
    assert np.array_equal(bits(got), bits(g["f64_out"]))
    pix = ods.image(40, 2).astype(np.int32)  # other dtypes widen to f64 like astype
    assert np.array_equal(bits(convolve_rows(pix, k, 3, 30)), bits(oconv.rows(pix, k.weights, 3, 30)))


@pytest.mark.parametrize("workers", [1, 3])
def test_host_bilateral_golden(workers):
    g = golden("bilateral")
    for i in range(4):
        side, seed, radius, ss, sr = g[f"meta_{i}"]
        lut = build_bilateral_lut(int(radius), float(ss), float(sr))
        img = g[f"img_{i}"]
        assert np.array_equal(bits(bilateral_rows(img, lut, 0, int(side), workers)), bits(g[f"out_{i}"])), i
        s3 = int(side) // 3
        assert np.array_equal(bits(bilateral_rows(img, lut, s3, s3 + 5, workers)), bits(g[f"strip_{i}"]))
    sp, rg = obil.lut(2, 1.5, 20.0)
    pix = ods.image(30, 6)
    assert np.array_equal(bits(bilateral_rows(pix, build_bilateral_lut(2, 1.5, 20.0), 7, 19)),
                          bits(obil.rows(pix, sp, rg, 2, 7, 19)))


class _SleepWorkload:
    """Both sides on the host, A twice as slow per unit as B: the measured
    calibration must land near fraction_a = 1/3."""

    name, unit = "toy", "units"

    def __init__(self, n=3000):
        self.n = n

    def partition(self, f):
        s = int(f * self.n)
        return (0, s), (s, self.n)

    def work_units(self, part):
        return float(part[1] - part[0])

    def run_part(self, device, part):
        import time

        rate = 1.0e5 if device.id.name == "A" else 2.0e5
        time.sleep((part[1] - part[0]) / rate)
        return part

    def merge(self, parts):
        return parts


def test_measured_calibration_finds_the_balanced_split():
    from paper_1303_2171_b200.worksharing import ShareOrigin, calibrate_measured

    share = calibrate_measured(_SleepWorkload(), Platform.build(1.0, 1.0), max_refinements=6)
    assert share.origin is ShareOrigin.CALIBRATED
    assert abs(share.fraction_a - 1 / 3) < 0.06, share.fraction_a
    assert share.probe.t_device_a > share.probe.t_device_b


def test_host_empty_shapes_and_dtypes():
    import numpy as np

    from paper_1303_2171_b200.gpu import host_empty

    for shape, dt in [(5, np.int64), ((3, 4), np.float64), ((0,), np.uint32), (1 << 21, np.float32)]:
        a = host_empty(shape, dt)
        assert a.dtype == np.dtype(dt) and a.shape == ((shape,) if isinstance(shape, int) else shape)
        assert a.flags.c_contiguous and a.flags.writeable


@pytest.mark.parametrize("idx", [np.int32, np.int64])
def test_host_spmv_rows_nnz_balanced_and_perm_scatter(idx):
    """Rows long enough for the threaded, nnz-balanced path (skewed row
    lengths, as in the nnz-sorted matrix), plain and with the fused
    y[perm[r]] scatter, against the oracle."""
    from oracle import spmv as ospmv

    rng = np.random.default_rng(5)
    rows = 20_000
    lens = np.sort(rng.zipf(1.6, rows).clip(0, 3000))[::-1]  # heavy rows first
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(idx)
    col = np.concatenate([np.sort(rng.choice(rows, int(k), replace=False)) for k in lens]).astype(idx)
    val = rng.standard_normal(int(ptr[-1]))
    x = rng.standard_normal(rows)
    assert ptr[-1] > 1 << 16
    m = CsrMatrix(rows, rows, ptr, col, val)
    want = ospmv.range_matvec(ptr.astype(np.int64), col.astype(np.int64), val, x, 0, rows)
    for w in (1, 3, 16):
        assert np.array_equal(bits(_host_range_matvec(m, x, 0, rows, w)), bits(want))
        assert np.array_equal(bits(_host_range_matvec(m, x, 777, 15_000, w)), bits(want[777:15_000]))
        perm = rng.permutation(rows).astype(idx)
        y = np.full(rows, np.nan)
        _host_range_matvec(m, x, 100, 19_000, w, perm=perm, y=y)
        assert np.array_equal(bits(y[perm[100:19_000]]), bits(want[100:19_000]))
        assert np.isnan(np.delete(y, perm[100:19_000])).all()


@pytest.mark.parametrize("workers", [1, 2, 15])
def test_host_histogram_many_tasks(workers):
    """Inputs large enough to be split into many dynamically claimed tasks
    (>= 2^18 elements each, up to 16 per worker), with per-task tables capped
    for wide bin counts: identical to np.bincount, and a bad element in the
    last task still raises."""
    rng = np.random.default_rng(11)
    data = rng.integers(0, 256, size=(1 << 24) + 12345, dtype=np.uint8)
    assert np.array_equal(host_histogram(data, 256, workers), np.bincount(data, minlength=256))
    wide = rng.integers(0, 1 << 20, size=(1 << 22) + 7, dtype=np.uint32)
    assert np.array_equal(host_histogram(wide, 1 << 20, workers), np.bincount(wide, minlength=1 << 20))
    bad = data.astype(np.int16)
    bad[-1] = 300
    with pytest.raises(ValueError):
        host_histogram(bad, 256, workers)


def test_result_pool_bookkeeping():
    """gpu._ResultPool (host_empty's pinned-result policy) on its own, no GPU:
    releases queue lock-free and are settled on the next booking; a release
    counts as a drop of its size class, and a pinned one frees its block."""
    from paper_1303_2171_b200.gpu import _ResultPool

    pool = _ResultPool()
    c = 1 << 25
    with pool.lock:
        pool.live[1] = (c, None, False)
        pool.live[2] = (c, None, True)
    pool.released(1)
    pool.released(2)  # finalizers: queued only
    assert len(pool.live) == 2 and pool.dropped == {} and pool.free == {}
    with pool.lock:
        pool.book()
    assert pool.live == {} and pool.dropped == {c: 2} and pool.free == {c: 1}
