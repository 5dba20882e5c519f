"""Histogram GPU parity: the drop-in (kernels_regular) vs the oracle and the
reference's golden outputs, through the C ABI.  Mirrors the reference's
tests/test_kernels_regular.py:32-67 and test_worksharing.py:139-184."""

import numpy as np
import pytest

from conftest import golden
from oracle import datasets as ods
from oracle import hist as ohist
from paper_1303_2171_b200 import _lib
from paper_1303_2171_b200.kernels_regular import HistogramWorkload, gpu_histogram, hybrid_histogram
from paper_1303_2171_b200.platform import DeviceId, Platform
from paper_1303_2171_b200.worksharing import WorkShare, formula_share, run_workshared

pytestmark = pytest.mark.gpu
SHARES = [i / 10 for i in range(11)]


def test_golden_all_shares(platform13):
    g = golden("hist")
    for i in range(4):
        n, seed, bins = (int(v) for v in g[f"meta_{i}"])
        data = ods.hist_values(n, seed, bins)
        for j, share in enumerate(SHARES):
            got = hybrid_histogram(data, bins, platform13, WorkShare.manual(share)).bins
            assert np.array_equal(got, g[f"bins_{i}"][j])
        # uint8 storage of the same values through the fast path
        got8 = hybrid_histogram(data.astype(np.uint8), bins, platform13, WorkShare.manual(0.0)).bins
        assert np.array_equal(got8, g[f"bins_{i}"][0])


def test_all_equal_adversary(platform13):
    data = np.full(1000, 7, dtype=np.int64)
    r = hybrid_histogram(data, 16, platform13)
    assert r.bins[7] == 1000 and r.bins.sum() == 1000 and np.count_nonzero(r.bins) == 1
    big = np.full((1 << 24) + 13, 200, dtype=np.uint8)
    assert gpu_histogram(big, 256)[200] == big.size


@pytest.mark.parametrize("dtype", [np.uint8, np.int8, np.uint16, np.int16, np.uint32, np.int32, np.uint64, np.int64])
def test_dtypes_and_ragged_offsets(dtype):
    base = ods.hist_values(100_000, 5, 100).astype(dtype)
    for off in (0, 1, 3, 7, 15):
        for tail in (0, 1, 9):
            part = base[off : base.size - tail]
            assert np.array_equal(gpu_histogram(part, 100), np.bincount(part.astype(np.int64), minlength=100))


def test_empty_and_tiny():
    assert np.array_equal(gpu_histogram(np.zeros(0, np.uint8), 256), np.zeros(256, np.int64))
    assert np.array_equal(gpu_histogram(np.array([3], np.uint8), 4), [0, 0, 0, 1])


def test_domain_errors_raise_value_error():
    with pytest.raises(ValueError):
        HistogramWorkload(np.array([0, 5, 256]), 256)
    with pytest.raises(ValueError):
        HistogramWorkload(np.array([-1]), 4)
    with pytest.raises(ValueError):  # uint8 above bin_count, caught on the device
        gpu_histogram(np.array([1, 2, 250], np.uint8), 200)
    with pytest.raises(ValueError):
        gpu_histogram(np.array([1, -2], np.int32), 200)


def test_many_bins_path():
    data = ods.hist_values(300_000, 9, 5000)
    assert np.array_equal(gpu_histogram(data, 5000), np.bincount(data, minlength=5000))


def test_device_resident_and_async():
    import torch

    data = ods.hist_values(1_000_003, 42, 256).astype(np.uint8)
    x = torch.from_numpy(data).cuda()
    out = torch.zeros(256, dtype=torch.int64, device="cuda")
    gpu_histogram(x, 256, out, asynchronous=True)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), np.bincount(data, minlength=256))


def test_device_generator_matches_reference_stream():
    import torch

    from paper_1303_2171_b200.rng import device_splitmix
    from oracle import rng as orng

    x = torch.empty(5000, dtype=torch.uint8, device="cuda")
    device_splitmix(x, 42, _lib.HB_GEN_LOW8, k0=1000)
    assert np.array_equal(x.cpu().numpy(), (orng.draws(42, 5000, first=1001) & np.uint64(255)).astype(np.uint8))
    y = torch.empty(777, dtype=torch.int64, device="cuda")
    device_splitmix(y, 7, _lib.HB_GEN_RAW)
    assert np.array_equal(y.cpu().numpy().view(np.uint64), orng.draws(7, 777))


def test_run_workshared_measured_and_modeled(platform13):
    from paper_1303_2171_b200.platform import Accounting, Platform

    data = ods.hist_values(1_000_000, 42)
    workload = HistogramWorkload(data, 256)
    result, report = run_workshared(platform13, workload, WorkShare.manual(0.25))
    assert np.array_equal(result.bins, np.bincount(data, minlength=256))
    assert report.gain_percent == pytest.approx(25.0, abs=1e-9)
    meas = Platform.build(1.0, 3.0, accounting=Accounting.MEASURED)
    result, report = run_workshared(meas, workload, formula_share(meas))
    assert np.array_equal(result.bins, np.bincount(data, minlength=256))
    assert report.timeline.busy(DeviceId.B) > 0


def test_measured_calibration_host_vs_gpu():
    # the share measured on this box (native host threads vs B200)
    from paper_1303_2171_b200.worksharing import calibrate_measured

    data = ods.hist_values(1 << 24, 5, 256).astype(np.uint8)
    p = Platform.build(1.0, 3.0)
    wl = HistogramWorkload(data, 256)
    share = calibrate_measured(wl, p, max_refinements=4)
    assert 0.0 <= share.fraction_a <= 1.0 and share.origin.value == "calibrated"
    assert share.probe.t_device_a > 0 and share.probe.t_device_b > 0 and len(share.probe.refinement_steps) >= 5
    out = hybrid_histogram(data, 256, p, share)
    assert np.array_equal(out.bins, np.bincount(data, minlength=256))
