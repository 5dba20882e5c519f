"""Column-ordered rounds SpMV plan (hb_spmv_plan_*, csrc/spmv_cor.cu): the
default bit-exact kernel for device int32 matrices.  Every case is compared
bit for bit with the oracle's restatement of the reference's row sums
(_csr_range_matvec, kernels_irregular.py:206-211) and with the SELL-32
kernel it replaces."""

import numpy as np
import pytest

from oracle import datasets as ods
from oracle import spmv as ospmv
from paper_1303_2171_b200.kernels_irregular import CsrMatrix, gpu_spmv, spmv_plan, spmv_preprocess
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def random_csr(rows, cols, max_len, seed, empty_frac=0.0):
    """Vectorised random CSR: row lengths U{0..max_len} (some rows emptied),
    strictly increasing columns per row."""
    rng = np.random.default_rng(seed)
    draw = np.sort(rng.integers(0, cols, size=(rows, max_len)), axis=1)
    keep = np.ones_like(draw, dtype=bool)
    keep[:, 1:] = np.diff(draw, axis=1) != 0
    keep &= np.arange(max_len)[None, :] < rng.integers(1, max_len + 1, size=rows)[:, None]
    keep[rng.random(rows) < empty_frac] = False
    lens = keep.sum(axis=1)
    ptr = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    return ptr, draw[keep].astype(np.int64), rng.uniform(-1.0, 1.0, size=int(ptr[-1])), rng.standard_normal(cols)


@pytest.mark.parametrize("rows,cols,max_len", [(1, 7, 3), (33, 100, 9), (147, 1_000, 12), (5_003, 20_000, 31),
                                               (70_001, 70_001, 31)])
def test_plan_bit_exact_row_ranges_and_perms(rows, cols, max_len):
    import torch

    ptr, col, val, x = random_csr(rows, cols, max_len, rows, empty_frac=0.1)
    want = ospmv.range_matvec(ptr, col, val, x, 0, rows)
    xd = torch.from_numpy(x).cuda()
    m = CsrMatrix(rows, cols, ptr, col, val)
    md = m.to_device(np.int32)
    for r0, r1 in ((0, rows), (rows // 3, rows), (min(5, rows), min(37, rows)), (rows - 1, rows)):
        if r1 == r0:
            continue
        plan = spmv_plan(md, r0, r1)
        assert plan.handle is not None, plan.reason
        assert plan.ctas <= r1 - r0 and plan.rounds * 1024 >= plan.nnz
        got = gpu_spmv(md, xd, r0, r1).cpu().numpy()
        sell = gpu_spmv(md, xd, r0, r1, method="exact_sell").cpu().numpy()
        assert np.array_equal(bits(got), bits(want[r0:r1])), (rows, r0, r1)
        assert np.array_equal(bits(got), bits(sell))
    prep = spmv_preprocess(m.to_device(), Platform.build(1.0, 3.0), WorkShare.manual(0.0))
    for pt in (prep.perm, prep.perm.to(torch.int64)):
        y = gpu_spmv(prep.permuted, xd, 0, rows, perm=pt).cpu().numpy()
        assert np.array_equal(bits(y), bits(want)), pt.dtype


def test_plan_golden_generator_matrix():
    """The reference generator's matrix (gen_csr stream, seed 42) through the
    public spmv_hybrid path: plan kernel == oracle bits."""
    import torch

    from oracle import rng as orng
    from paper_1303_2171_b200.kernels_irregular import spmv_hybrid

    rows = 20_000
    ptr, col, val = ods.csr(rows, rows, 42, 8e-4)
    x = 2.0 * orng.uniform_floats(orng.mix_seed(42, 0xDEC0), rows) - 1.0
    prep = spmv_preprocess(CsrMatrix(rows, rows, ptr, col, val).to_device(), Platform.build(1.0, 3.0),
                           WorkShare.manual(0.0))
    y = spmv_hybrid(prep, torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(bits(y), bits(ospmv.range_matvec(ptr, col, val, x, 0, rows)))
    assert spmv_plan(prep.permuted, 0, rows).handle is not None


def test_plan_several_chunks():
    """More rows than one CTA per SM holds (8192 each): the range is cut into
    chunks that run one after the other."""
    import torch

    rows = 1_400_000
    ptr, col, val, x = random_csr(rows, 300_000, 4, 7, empty_frac=0.05)
    md = CsrMatrix(rows, 300_000, ptr, col, val).to_device(np.int32)
    plan = spmv_plan(md, 0, rows)
    assert plan.handle is not None and plan.chunks >= 2, (plan.chunks, plan.reason)
    got = gpu_spmv(md, torch.from_numpy(x).cuda(), 0, rows).cpu().numpy()
    assert np.array_equal(bits(got), bits(ospmv.range_matvec(ptr, col, val, x, 0, rows)))


def test_plan_falls_back_on_a_very_long_row():
    """A row with far more nonzeros than the scheduler's round window: no
    plan (reason given), the SELL kernel answers, still bit-exact."""
    import torch

    rng = np.random.default_rng(3)
    cols = 400_000
    long_cols = np.sort(rng.choice(cols, size=200_000, replace=False))
    ptr = np.array([0, 200_000, 200_002, 200_003], dtype=np.int64)
    col = np.concatenate([long_cols, [5, 9], [17]]).astype(np.int64)
    val = rng.uniform(-1, 1, size=col.size)
    x = rng.standard_normal(cols)
    md = CsrMatrix(3, cols, ptr, col, val).to_device(np.int32)
    plan = spmv_plan(md, 0, 3)
    assert plan.handle is None and plan.reason
    got = gpu_spmv(md, torch.from_numpy(x).cuda(), 0, 3).cpu().numpy()
    assert np.array_equal(bits(got), bits(ospmv.sequential_rows(ptr, col, val, x)))


def test_plan_zero_nonzeros():
    import torch

    ptr = np.zeros(11, dtype=np.int64)
    md = CsrMatrix(10, 4, ptr, np.zeros(0, np.int64), np.zeros(0)).to_device(np.int32)
    y = gpu_spmv(md, torch.ones(4, dtype=torch.float64).cuda(), 0, 10).cpu().numpy()
    assert np.array_equal(bits(y), bits(np.zeros(10)))
