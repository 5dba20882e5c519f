"""Sort GPU parity: bit-exact sorted output (= the reference's, the sorted
multiset being unique), stable payload, and the reference's work accounting;
mirrors tests/test_kernels_regular.py:73-120 and acceptance :126-132."""

import numpy as np
import pytest

from conftest import golden
from oracle import datasets as ods
from oracle import sort as osort
from paper_1303_2171_b200.kernels_regular import gpu_sort, hybrid_sort, sample_sort_hybrid
from paper_1303_2171_b200.worksharing import WorkShare

pytestmark = pytest.mark.gpu
SHARES = [i / 10 for i in range(11)]


@pytest.mark.parametrize("name", ["uar50k", "dups", "rev", "tiny", "const"])
def test_golden_work_accounting(platform13, name):
    g = golden("sort")
    data = g[f"{name}_data"]
    for sh, wa, wb in g[f"{name}_work"]:
        share = None if sh < 0 else WorkShare.manual(float(sh))
        out, got_a, got_b = sample_sort_hybrid(data, platform13, share=share)
        assert np.array_equal(out, np.sort(data))
        assert (got_a, got_b) == (wa, wb)


def test_reference_unit_cases(platform13):
    assert np.array_equal(hybrid_sort(np.arange(1000), platform13), np.arange(1000))
    assert np.array_equal(hybrid_sort(np.arange(1000)[::-1].copy(), platform13), np.arange(1000))
    d = ods.sort_keys(100_000, 42) % 5000
    assert np.array_equal(hybrid_sort(d, platform13), np.sort(d))
    assert np.array_equal(hybrid_sort(np.array([3]), platform13), [3])
    assert np.array_equal(hybrid_sort(np.full(5000, 9), platform13), np.full(5000, 9))
    assert hybrid_sort(np.array([], dtype=np.int64), platform13).size == 0
    with pytest.raises(ValueError):
        hybrid_sort(np.arange(10), platform13, leaf_a=4, leaf_b=8)
    _, wa, wb = sample_sort_hybrid(ods.sort_keys(50_000, 1), platform13)
    assert wa + wb == 50_000 and wa / 50_000 == pytest.approx(0.25, abs=0.02)


def test_split_invariance(platform13):
    data = ods.sort_keys(3000, 2)
    for share in SHARES:
        assert np.array_equal(hybrid_sort(data, platform13, share=WorkShare.manual(share)), np.sort(data))
    for seed in range(20, 25):
        data = ods.sort_keys(1200, seed)
        for share in (0.0, 0.3, 0.7):
            assert np.array_equal(hybrid_sort(data, platform13, share=WorkShare.manual(share)), np.sort(data))


@pytest.mark.parametrize("dtype", [np.uint32, np.int32, np.uint64, np.int64])
@pytest.mark.parametrize("n", [2, 6143, 6144, 6145, 4095, 4097, 1_000_003])
def test_gpu_sort_types_sizes_stable(dtype, n):
    raw = ods.sort_keys(n, n) if n > 0 else np.zeros(0, np.int64)
    if np.dtype(dtype).kind == "i":
        keys = (raw - (1 << 31)).astype(dtype)  # negatives too
    else:
        keys = raw.astype(dtype)
    keys = keys % np.array(977, dtype=dtype) if n > 10_000 else keys  # many ties at large n
    if np.dtype(dtype).itemsize == 8:
        keys = keys * np.array(1 << 20, dtype=dtype)  # exercise the high digits
    pay = np.arange(n, dtype=np.uint32)
    k, p, _ = gpu_sort(keys, pay)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(k, keys[order])
    assert np.array_equal(p, order.astype(np.uint32))
    assert osort.check_stable_payload(keys, k, p)


def test_gpu_sort_skewed_and_pass_skipping():
    n = 300_000
    keys = np.zeros(n, dtype=np.uint32)
    keys[::1000] = 7  # two distinct values → a single live digit pass
    k, _, passes = gpu_sort(keys)
    assert np.array_equal(k, np.sort(keys)) and passes == 1
    k, _, passes = gpu_sort(np.full(n, 12345, dtype=np.int64))
    assert passes == 0 and np.all(k == 12345)
    hi = (ods.sort_keys(n, 5) << 32).astype(np.int64)  # only the high 4 digits live
    k, _, passes = gpu_sort(hi)
    assert np.array_equal(k, np.sort(hi)) and passes == 4


def test_device_resident_in_place():
    import torch

    keys = ods.sort_keys(2_000_001, 42).astype(np.uint32)
    kt = torch.from_numpy(keys.view(np.int32)).cuda()
    vt = torch.arange(keys.size, dtype=torch.int32, device="cuda")
    # view the int32 storage as uint32 keys through the C ABI
    from paper_1303_2171_b200 import _lib
    from paper_1303_2171_b200.gpu import current_stream_handle, vp

    _lib.call("hb_sort", vp(kt.data_ptr()), vp(kt.data_ptr()), 5, vp(vt.data_ptr()), vp(vt.data_ptr()),
              keys.size, None, _lib.HB_DEVICE_PTRS, current_stream_handle(kt))
    got_k = kt.cpu().numpy().view(np.uint32)
    got_v = vt.cpu().numpy()
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(got_k, keys[order]) and np.array_equal(got_v, order)


def test_split_points_kernel():
    import torch

    from paper_1303_2171_b200.sort_exchange import gpu_split_points, host_split_points

    keys = np.sort(ods.sort_keys(100_000, 4) % 1000).astype(np.int64)
    idx = np.arange(keys.size, dtype=np.int32)
    pk = np.array([0, 5, 500, 999, 2000], dtype=np.int64)
    pi = np.array([0, 40_000, 50_000, 99_999, 0], dtype=np.int32)
    want = host_split_points(*(torch.from_numpy(a) for a in (keys, idx, pk, pi)))
    got = gpu_split_points(*(torch.from_numpy(a).cuda() for a in (keys, idx, pk, pi)))
    assert want.tolist() == got.cpu().tolist()


@pytest.mark.parametrize("ballot", [False, True])
@pytest.mark.parametrize("dtype", [np.uint32, np.int32, np.uint64, np.int64])
def test_stable_payload_adversarial_duplicates(ballot, dtype):
    """The production ranking (lane-ordered shared atomics, device-checked)
    and the ballot multi-split both give the stable argsort on inputs built
    to stress the ranking: all-equal, two values alternating, runs of 32
    equal keys per warp, one hot digit among random keys, and every digit
    position constant but one."""
    from oracle import sort as osort
    from paper_1303_2171_b200.kernels_regular import gpu_sort

    rs = np.random.default_rng(11)
    n = 3_000_017
    cases = {
        "all_equal": np.full(n, 7, dtype=np.int64),
        "alternating": np.arange(n) % 2,
        "warp_runs": (np.arange(n) // 32) % 5,
        "hot_digit": np.where(rs.random(n) < 0.9, 42, rs.integers(0, 1 << 30, n)),
        "one_live_digit": (rs.integers(0, 256, n) << 16) | 0x1234,
        "few_values": rs.integers(0, 3, n),
    }
    for name, raw in cases.items():
        keys = raw.astype(dtype)
        pay = np.arange(n, dtype=np.uint32)
        k, v, _ = gpu_sort(keys, pay, ballot=ballot)
        assert np.array_equal(k, np.sort(keys, kind="stable")), name
        assert osort.check_stable_payload(keys, k, v), name
        import torch

        kt = torch.from_numpy(keys.view(np.int64 if keys.itemsize == 8 else np.int32)).cuda()
        kt = kt.view(getattr(torch, np.dtype(dtype).name))
        vt = torch.arange(n, dtype=torch.int32, device="cuda")
        gpu_sort(kt, vt, ballot=ballot)  # device-resident, in place
        got_v = vt.cpu().numpy().astype(np.uint32)
        assert np.array_equal(got_v, v), name
