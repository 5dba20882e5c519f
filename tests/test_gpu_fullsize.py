"""BASELINE.json full sizes on one B200, checked through size-independent
properties (the oracle cannot run these sizes in seconds): bit-exact
histogram against an independent count, sort order + stable-argsort payload,
list ranks as distances along succ, bit-exact SpMV at 1M rows, filter strips
against the oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_histogram_2e30_u8():
    import torch

    from paper_1303_2171_b200 import _lib
    from paper_1303_2171_b200.kernels_regular import gpu_histogram
    from paper_1303_2171_b200.rng import device_splitmix

    n = 1 << 30
    x = torch.empty(n, dtype=torch.uint8, device="cuda")
    device_splitmix(x, 42, _lib.HB_GEN_LOW8)
    got = gpu_histogram(x, 256)
    want = torch.bincount(x.to(torch.int32), minlength=256)  # independent count (chunk-free)
    assert torch.equal(got.cpu(), want.cpu().to(torch.int64)) and int(got.sum()) == n


def test_sort_2e28_u32_with_stable_payload():
    import torch

    from paper_1303_2171_b200 import _lib
    from paper_1303_2171_b200.kernels_regular import gpu_sort
    from paper_1303_2171_b200.rng import device_splitmix

    n = 1 << 28
    keys = torch.empty(n, dtype=torch.int32, device="cuda")
    device_splitmix(keys, 42, _lib.HB_GEN_HI32)
    keys_in = keys.clone()
    vals = torch.arange(n, dtype=torch.int32, device="cuda")
    gpu_sort(keys.view(torch.uint32), vals.view(torch.uint32))
    u = keys.to(torch.int64) & 0xFFFFFFFF  # unsigned order
    d = u[1:] - u[:-1]
    assert bool((d >= 0).all())
    p = vals.to(torch.int64)
    assert torch.equal(torch.bincount(p, minlength=n), torch.ones(n, dtype=torch.int64, device="cuda"))
    assert torch.equal(keys_in[p], keys)  # payload = a permutation taking input to output
    assert bool(((d > 0) | (p[1:] > p[:-1])).all())  # stable: equal keys keep input order


def test_list_ranking_2e28():
    import torch

    from paper_1303_2171_b200.datasets import device_gen_list
    from paper_1303_2171_b200.kernels_irregular import gpu_list_rank

    n = 1 << 28
    succ, head = device_gen_list(n, 42)
    rank = gpu_list_rank(succ, head)
    s = succ.to(torch.int64)
    assert int(rank[head]) == 0
    nxt = s >= 0
    assert bool((rank[s[nxt]] == rank[nxt] + 1).all())  # one step along succ = one rank
    assert int(rank.max()) == n - 1 and int((~nxt).sum()) == 1


def test_spmv_1m_bit_exact():
    import torch

    from oracle import spmv as ospmv
    from paper_1303_2171_b200.datasets import csr_arrays
    from paper_1303_2171_b200.kernels_irregular import CsrMatrix, gpu_spmv, spmv_preprocess
    from paper_1303_2171_b200.platform import Platform
    from paper_1303_2171_b200.rng import mix_seed, uniform_floats
    from paper_1303_2171_b200.worksharing import WorkShare

    rows = 1_000_000
    ptr, col, val = csr_arrays(rows, rows, 42, 1.6e-5)
    x = 2.0 * uniform_floats(mix_seed(42, 0xDEC0), rows) - 1.0
    prep = spmv_preprocess(CsrMatrix(rows, rows, ptr, col, val), Platform.build(1.0, 3.0), WorkShare.manual(0.0))
    dm = prep.permuted.to_device(np.int32)
    perm = torch.from_numpy(np.asarray(prep.perm, dtype=np.int32)).cuda()
    y = torch.empty(rows, dtype=torch.float64, device="cuda")
    gpu_spmv(dm, torch.from_numpy(x).cuda(), 0, rows, y=y, perm=perm)
    p = prep.permuted
    want = ospmv.hybrid(prep.perm, (p.row_ptr, p.col_idx, p.values), 0, x)
    assert np.array_equal(y.cpu().numpy().view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("kind", ["bilat", "conv"])
def test_filters_16384_strips(kind):
    import torch

    from oracle import bilateral as obil
    from oracle import conv as oconv
    from paper_1303_2171_b200.datasets import device_gen_image
    from paper_1303_2171_b200.kernels_regular import (
        FilterKernel,
        build_bilateral_lut,
        gpu_bilateral_rows,
        gpu_convolve_rows,
    )

    side = 16384
    img = device_gen_image(side, 42)
    host = img.cpu().numpy()
    if kind == "bilat":
        lut = build_bilateral_lut(5, 2.5, 40.0)
        out = gpu_bilateral_rows(img, lut, 0, side)
        sp, rg = obil.lut(5, 2.5, 40.0)
        ref = lambda a, b: obil.rows(host, sp, rg, 5, a, b)  # noqa: E731
    else:
        k = FilterKernel.gaussian(7)
        out = gpu_convolve_rows(img, k, 0, side)
        ref = lambda a, b: oconv.rows(host, k.weights, a, b)  # noqa: E731
    for a, b in [(0, 9), (8190, 8200), (side - 9, side)]:
        got = out[a:b].cpu().numpy()
        assert np.array_equal(got.view(np.uint64), ref(a, b).view(np.uint64)), (kind, a)
    del out
    torch.cuda.empty_cache()
