"""SpMV GPU parity through the C ABI: bit-exact against the reference's own
outputs (golden) and the oracle's sequential row sums; mirrors the
reference's tests/test_kernels_irregular.py:70-128 and acceptance :153-160."""

import numpy as np
import pytest

from conftest import golden
from oracle import datasets as ods
from oracle import rng as orng
from oracle import spmv as ospmv
from paper_1303_2171_b200.errors import StructuralError
from paper_1303_2171_b200.kernels_irregular import (
    CsrMatrix,
    SpmvPrep,
    SpmvWorkload,
    gpu_spmv,
    spmv_hybrid,
    spmv_preprocess,
)
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare, run_workshared

pytestmark = pytest.mark.gpu
SHARES = [i / 10 for i in range(11)]


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def test_golden_bit_exact_all_shares(platform13):
    g = golden("spmv")
    for i in range(4):
        m = CsrMatrix(len(g[f"ptr_{i}"]) - 1, len(g[f"x_{i}"]), g[f"ptr_{i}"], g[f"col_{i}"], g[f"val_{i}"])
        x = g[f"x_{i}"]
        prep = spmv_preprocess(m, platform13)
        assert np.array_equal(prep.perm, g[f"perm_{i}"]) and prep.split_row == g[f"split_{i}"][0]
        assert np.array_equal(bits(spmv_hybrid(prep, x)), bits(g[f"y_{i}"]))
        for j, sh in enumerate(SHARES):
            p = spmv_preprocess(m, platform13, WorkShare.manual(sh))
            assert p.split_row == g[f"split_{i}"][j + 1]
            assert np.array_equal(bits(spmv_hybrid(p, x)), bits(g[f"y_{i}"]))
        # device-resident matrix and x, fused un-permute
        dprep = spmv_preprocess(m.to_device(), platform13, WorkShare.manual(0.0))
        import torch

        xd = torch.from_numpy(x).cuda()
        assert np.array_equal(dprep.perm.cpu().numpy(), g[f"perm_{i}"])  # device spmv_preprocess
        y = gpu_spmv(dprep.permuted, xd, 0, m.rows, perm=dprep.perm)
        assert np.array_equal(bits(y.cpu().numpy()), bits(g[f"y_{i}"]))


def test_every_split_row_sound(platform13):
    ptr, col, val = ods.csr(30, 30, 5, 0.15)
    m = CsrMatrix(30, 30, ptr, col, val)
    x = orng.uniform_floats(99, 30)
    base = spmv_preprocess(m, platform13)
    want = ospmv.hybrid(base.perm, (base.permuted.row_ptr, base.permuted.col_idx, base.permuted.values), 0, x)
    for split in range(0, 31):
        prep = SpmvPrep(base.permuted, base.perm, split)
        assert np.array_equal(bits(spmv_hybrid(prep, x)), bits(want))


def test_kats_identity_zero_and_mismatch(platform13):
    prep = spmv_preprocess(CsrMatrix.identity(3), platform13)
    assert np.array_equal(spmv_hybrid(prep, np.array([1.0, 2.0, 3.0])), [1.0, 2.0, 3.0])
    zero = CsrMatrix(3, 3, np.zeros(4, dtype=np.int64), np.zeros(0, np.int64), np.zeros(0))
    assert np.array_equal(spmv_hybrid(spmv_preprocess(zero, platform13), np.ones(3)), np.zeros(3))
    with pytest.raises(ValueError):
        spmv_hybrid(prep, np.ones(4))


@pytest.mark.parametrize("idx", [np.int32, np.int64])
def test_long_and_empty_rows_bit_exact(idx):
    # rows far longer than one staged chunk, interleaved with empty rows
    rng = np.random.default_rng(3)
    lens = np.array([0, 5, 0, 9000, 1, 0, 20000, 3, 0, 0, 4097, 4096, 4095, 17])
    rows, cols = lens.size, 50_000
    ptr = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    col = np.concatenate([np.sort(rng.choice(cols, k, replace=False)) for k in lens]).astype(np.int64)
    val = rng.standard_normal(ptr[-1])
    x = rng.standard_normal(cols)
    m = CsrMatrix(rows, cols, ptr, col, val)
    want = ospmv.sequential_rows(ptr, col, val, x)
    assert np.array_equal(bits(gpu_spmv(m, x, 0, rows)), bits(want))
    md = m.to_device(idx)
    import torch

    got = gpu_spmv(md, torch.from_numpy(x).cuda(), 0, rows)
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))
    got = gpu_spmv(md, torch.from_numpy(x).cuda(), 2, 9)
    assert np.array_equal(bits(got.cpu().numpy()), bits(want[2:9]))


def test_int32_row_ranges_and_unaligned_views_bit_exact():
    # lane-per-row kernel: many tiles, row ranges that start/end inside a tile,
    # and col/val views whose first element is not 16-byte aligned
    import torch

    ptr, col, val = ods.csr(30_011, 30_011, 7, 6e-4)
    x = 2.0 * orng.uniform_floats(orng.mix_seed(7, 0xDEC0), 30_011) - 1.0
    want = ospmv.sequential_rows(ptr, col, val, x)
    m = CsrMatrix(30_011, 30_011, ptr, col, val)
    md = m.to_device(np.int32)
    xd = torch.from_numpy(x).cuda()
    for r0, r1 in [(0, 30_011), (1, 30_011), (5, 37), (31, 33), (12_345, 29_999), (30_010, 30_011)]:
        got = gpu_spmv(md, xd, r0, r1)
        assert np.array_equal(bits(got.cpu().numpy()), bits(want[r0:r1])), (r0, r1)
    # views offset by 1..3 elements: the bulk copies start mid 16-byte block
    pt = torch.from_numpy(ptr.astype(np.int32)).cuda()
    for shift in (1, 2, 3):
        ct = torch.cat([torch.zeros(shift, dtype=torch.int32), torch.from_numpy(col.astype(np.int32))]).cuda()[shift:]
        vt = torch.cat([torch.zeros(shift, dtype=torch.float64), torch.from_numpy(val)]).cuda()[shift:]
        assert ct.data_ptr() % 16 != 0 or vt.data_ptr() % 16 != 0
        got = gpu_spmv(CsrMatrix(30_011, 30_011, pt, ct, vt), xd, 0, 30_011)
        assert np.array_equal(bits(got.cpu().numpy()), bits(want)), shift


def test_warp_mode_within_tolerance():
    ptr, col, val = ods.csr(20_000, 20_000, 42, 8e-4)
    x = 2.0 * orng.uniform_floats(orng.mix_seed(42, 0xDEC0), 20_000) - 1.0
    m = CsrMatrix(20_000, 20_000, ptr, col, val)
    want = ospmv.range_matvec(ptr, col, val, x, 0, 20_000)
    got = gpu_spmv(m, x, 0, 20_000, exact=False)
    assert np.allclose(got, want, rtol=1e-9, atol=1e-12)
    assert np.array_equal(bits(gpu_spmv(m, x, 0, 20_000)), bits(want))


def _power_law_csr(rows, cols, seed):
    # unsorted rows whose lengths span 0 .. 200k nnz (merge-path's case)
    rng = np.random.default_rng(seed)
    lens = np.minimum((rng.pareto(1.2, rows) * 3).astype(np.int64), cols)
    lens[rng.integers(0, rows, 3)] = [200_000, 50_000, 0]
    lens[::97] = 0
    ptr = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    col = np.concatenate([np.sort(rng.choice(cols, int(k), replace=False)) if k else np.zeros(0, np.int64)
                          for k in lens]).astype(np.int64)
    val = rng.standard_normal(int(ptr[-1]))
    return ptr, col, val


@pytest.mark.parametrize("idx", [np.int32, np.int64])
def test_merge_path_within_tolerance(idx):
    import torch

    rows, cols = 30_000, 250_000
    ptr, col, val = _power_law_csr(rows, cols, 5)
    x = np.random.default_rng(6).standard_normal(cols)
    want = ospmv.range_matvec(ptr, col, val, x, 0, rows)
    scale = np.abs(val).max() * np.abs(x).max()
    tol = dict(rtol=1e-9, atol=1e-12 * scale * np.sqrt(np.maximum(np.diff(ptr), 1)).max())
    m = CsrMatrix(rows, cols, ptr, col, val)
    assert np.allclose(gpu_spmv(m, x, 0, rows, method="merge"), want, **tol)
    md = m.to_device(idx)
    xd = torch.from_numpy(x).cuda()
    for r0, r1 in [(0, rows), (1, 2), (17, 9_000), (rows - 5, rows)]:
        got = gpu_spmv(md, xd, r0, r1, method="merge").cpu().numpy()
        assert np.allclose(got, want[r0:r1], **tol), (r0, r1)
    perm = torch.from_numpy(np.random.default_rng(1).permutation(rows).astype(np.int64)).cuda()
    y = torch.zeros(rows, dtype=torch.float64, device="cuda")
    gpu_spmv(md, xd, 0, rows, y=y, perm=perm, method="merge")
    yp = np.empty(rows)
    yp[perm.cpu().numpy()] = want
    assert np.allclose(y.cpu().numpy(), yp, **tol)


def test_device_csr_validation():
    import torch

    ptr = torch.tensor([0, 2, 1], dtype=torch.int64, device="cuda")
    with pytest.raises(StructuralError):
        CsrMatrix(2, 3, ptr, torch.tensor([0, 1], device="cuda"), torch.ones(2, dtype=torch.float64, device="cuda"))
    with pytest.raises(StructuralError):
        CsrMatrix(1, 3, torch.tensor([0, 2], device="cuda"), torch.tensor([2, 1], device="cuda"),
                  torch.ones(2, dtype=torch.float64, device="cuda"))
    with pytest.raises(StructuralError):
        CsrMatrix(1, 2, torch.tensor([0, 1], device="cuda"), torch.tensor([5], device="cuda"),
                  torch.ones(1, dtype=torch.float64, device="cuda"))
    ok = CsrMatrix(2, 3, torch.tensor([0, 1, 3], device="cuda"), torch.tensor([2, 0, 1], device="cuda"),
                   torch.ones(3, dtype=torch.float64, device="cuda"))
    assert ok.nnz == 3


def test_workshared_runner_path():
    from paper_1303_2171_b200.platform import Accounting

    ptr, col, val = ods.csr(5000, 5000, 42, 0.002)
    m = CsrMatrix(5000, 5000, ptr, col, val)
    x = 2.0 * orng.uniform_floats(orng.mix_seed(42, 0xDEC0), 5000) - 1.0
    plat = Platform.build(1.0, 3.0, accounting=Accounting.MEASURED)
    prep = spmv_preprocess(m, plat)
    wl = SpmvWorkload(prep, x)
    y, report = run_workshared(plat, wl, WorkShare.manual(0.25))
    perm, permuted, split = ospmv.preprocess(ptr, col, val, 1.0, 3.0, None)
    assert np.array_equal(bits(y), bits(ospmv.hybrid(perm, permuted, split, x)))
    assert report.pure_b_time > 0


def test_device_preprocess_matches_host(platform13):
    import torch

    g = golden("spmv")
    for i in range(4):
        m = CsrMatrix(len(g[f"ptr_{i}"]) - 1, len(g[f"x_{i}"]), g[f"ptr_{i}"], g[f"col_{i}"], g[f"val_{i}"])
        for share in (None, WorkShare.manual(0.0), WorkShare.manual(0.37)):
            hp = spmv_preprocess(m, platform13, share)
            dp = spmv_preprocess(m.to_device(np.int64), platform13, share)
            assert np.array_equal(np.asarray(dp.perm.cpu()), hp.perm) and dp.split_row == hp.split_row
            assert np.array_equal(dp.permuted.row_ptr.cpu().numpy(), hp.permuted.row_ptr)
            assert np.array_equal(dp.permuted.col_idx.cpu().numpy(), hp.permuted.col_idx)
            assert np.array_equal(dp.permuted.values.cpu().numpy(), hp.permuted.values)
    # larger, int32 indices, then a full device SpMV with the fused un-permute
    ptr, col, val = ods.csr(200_000, 200_000, 7, 8e-5)
    m = CsrMatrix(200_000, 200_000, ptr, col, val)
    x = 2.0 * orng.uniform_floats(orng.mix_seed(7, 0xDEC0), 200_000) - 1.0
    dp = spmv_preprocess(m.to_device(np.int32), platform13, WorkShare.manual(0.0))
    y = gpu_spmv(dp.permuted, torch.from_numpy(x).cuda(), 0, m.rows, perm=dp.perm)
    perm, permuted, split = ospmv.preprocess(ptr, col, val, 1.0, 3.0, 0.0)
    want = ospmv.hybrid(perm, permuted, split, x)
    assert np.array_equal(bits(y.cpu().numpy()), bits(want))


@pytest.mark.parametrize("pdt", [np.int32, np.int64])
def test_host_path_unpermute_from_stage(pdt):
    """Host arrays, multi-threaded un-permute out of the pinned stage: every
    row must land at y[perm[r]] bit-exactly and nothing else may be written,
    for full and partial ranges, int32 and int64 perms."""
    rows = 150_000
    ptr, col, val = ods.csr(rows, rows, 7, 4e-5)
    x = 2.0 * orng.uniform_floats(orng.mix_seed(7, 0xDEC0), rows) - 1.0
    m = CsrMatrix(rows, rows, ptr, col, val)
    want = ospmv.range_matvec(ptr, col, val, x, 0, rows)
    perm = np.random.default_rng(3).permutation(rows).astype(pdt)
    for r0, r1 in [(0, rows), (1234, 1234 + 70_000), (rows - 65_536, rows)]:
        y = np.full(rows, np.nan)
        gpu_spmv(m, x, r0, r1, y, perm)
        assert np.array_equal(bits(y[perm[r0:r1]]), bits(want[r0:r1]))
        assert np.isnan(np.delete(y, perm[r0:r1])).all()


def test_host_path_unpermute_beyond_one_pinned_stage():
    """> 4M rows: the row sums no longer fit one 32 MB pinned stage, so the
    call takes the device-buffer + staged D2H un-permute path."""
    rows = 4_300_000
    rng = np.random.default_rng(8)
    lens = rng.integers(0, 4, rows)
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col = rng.integers(0, rows, int(ptr[-1])).astype(np.int64)
    # columns strictly increasing per row (CSR invariant): sort within rows, drop repeats
    order = np.lexsort((col, np.repeat(np.arange(rows), lens)))
    col = col[order]
    keep = np.ones(col.size, bool)
    row_of = np.repeat(np.arange(rows), lens)
    keep[1:] = ~((row_of[1:] == row_of[:-1]) & (col[1:] == col[:-1]))
    col, row_of = col[keep], row_of[keep]
    ptr = np.concatenate([[0], np.cumsum(np.bincount(row_of, minlength=rows))]).astype(np.int64)
    val = rng.standard_normal(col.size)
    x = rng.standard_normal(rows)
    m = CsrMatrix(rows, rows, ptr, col, val)
    perm = rng.permutation(rows).astype(np.int64)
    y = np.full(rows, np.nan)
    gpu_spmv(m, x, 0, rows, y, perm)
    want = ospmv.range_matvec(ptr, col, val, x, 0, rows)
    assert np.array_equal(bits(y[perm]), bits(want))


def test_sell_layout_matches_csr_kernel_and_oracle():
    """The SELL-32 copy (default for device int32 matrices) and the CSR
    lane-per-row kernel give the same bits as the oracle's sequential sums:
    unsorted and nnz-sorted matrices, empty and long rows, row ranges that
    start and end inside a 32-row tile, y_perm slices and fused perm stores."""
    import torch

    from paper_1303_2171_b200.kernels_irregular import sell_layout

    rng = np.random.default_rng(21)
    for rows, cols, dens in ((1, 7, 0.5), (33, 100, 0.1), (5_003, 20_000, 1e-3), (70_001, 70_001, 2.5e-4)):
        ptr, col, val = ods.csr(rows, cols, rows, dens)
        lens = np.diff(ptr)
        lens[rng.random(rows) < 0.1] = 0  # empty rows
        keep = np.concatenate([np.arange(ptr[r], ptr[r] + lens[r]) for r in range(rows)]).astype(np.int64) \
            if lens.sum() else np.zeros(0, np.int64)
        ptr = np.zeros(rows + 1, dtype=np.int64)
        np.cumsum(lens, out=ptr[1:])
        col, val = col[keep], val[keep]
        x = rng.standard_normal(cols)
        want = ospmv.sequential_rows(ptr, col, val, x)
        for sort in (False, True):
            m = CsrMatrix(rows, cols, ptr, col, val)
            if sort:
                prep = spmv_preprocess(m.to_device(), Platform.build(1.0, 3.0), WorkShare.manual(0.0))
                md, perm = prep.permuted, prep.perm
            else:
                md, perm = m.to_device(np.int32), None
            xd = torch.from_numpy(x).cuda()
            toff, scol, sval = sell_layout(md)
            assert int(toff[-1]) == scol.numel() >= md.nnz
            for r0, r1 in ((0, rows), (rows // 3, rows), (min(5, rows), min(37, rows)), (rows - 1, rows)):
                a = gpu_spmv(md, xd, r0, r1)
                b = gpu_spmv(md, xd, r0, r1, method="exact_csr")
                assert np.array_equal(bits(a.cpu().numpy()), bits(b.cpu().numpy())), (rows, sort, r0, r1)
            if perm is not None:
                for pt in (perm, perm.to(torch.int64)):
                    y = gpu_spmv(md, xd, 0, rows, perm=pt)
                    assert np.array_equal(bits(y.cpu().numpy()), bits(want)), (rows, pt.dtype)
            else:
                assert np.array_equal(bits(gpu_spmv(md, xd, 0, rows).cpu().numpy()), bits(want)), rows
