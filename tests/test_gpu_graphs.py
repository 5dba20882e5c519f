"""The device-resident, asynchronous library calls are CUDA-graph capturable:
an iterative caller (the paper amortises spmv_preprocess over SpMV
iterations) can capture a step once and replay it.  Each
replay must reproduce the eager result bit for bit."""

import numpy as np
import pytest

from oracle import datasets as ods
from paper_1303_2171_b200.kernels_irregular import CsrMatrix, gpu_spmv, spmv_preprocess
from paper_1303_2171_b200.kernels_regular import (
    FilterKernel,
    build_bilateral_lut,
    gpu_bilateral_rows,
    gpu_convolve_rows,
    gpu_histogram,
    gpu_sort,
)
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

pytestmark = pytest.mark.gpu


def _capture(step):
    """Warm up eagerly, capture one call on a side stream, return the graph."""
    import torch

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
    torch.cuda.synchronize()
    return g


def _bits(t):
    import torch

    return t.contiguous().view(torch.uint8).cpu().numpy()


def test_spmv_and_histogram_replay():
    import torch

    rows = 50_000
    ptr, col, val = ods.csr(rows, rows, 42, 3e-4)
    prep = spmv_preprocess(CsrMatrix(rows, rows, ptr, col, val).to_device(), Platform.build(1.0, 3.0),
                           WorkShare.manual(0.0))
    x = torch.rand(rows, dtype=torch.float64, device="cuda")
    y = torch.empty(rows, dtype=torch.float64, device="cuda")
    eager = gpu_spmv(prep.permuted, x, 0, rows, perm=prep.perm).clone()
    g = _capture(lambda: gpu_spmv(prep.permuted, x, 0, rows, y=y, perm=prep.perm, asynchronous=True))
    for _ in range(3):
        y.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(_bits(y), _bits(eager))

    data = torch.randint(0, 256, (3_000_001,), dtype=torch.uint8, device="cuda")
    out = torch.empty(256, dtype=torch.int64, device="cuda")
    want = gpu_histogram(data, 256).cpu().numpy()
    g = _capture(lambda: gpu_histogram(data, 256, out, asynchronous=True))
    for _ in range(3):
        out.fill_(-1)
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), want)


def test_filters_replay():
    import torch

    rng = np.random.default_rng(5)
    img = torch.from_numpy(rng.integers(0, 256, size=(300, 257), dtype=np.uint8)).cuda()
    lut = build_bilateral_lut(3, 1.5, 30.0)
    kern = FilterKernel(rng.uniform(-1, 1, size=(5, 5)))
    for fn in (lambda o: gpu_bilateral_rows(img, lut, 7, 290, out=o, asynchronous=True),
               lambda o: gpu_convolve_rows(img, kern, 7, 290, out=o, asynchronous=True)):
        out = torch.empty((283, 257), dtype=torch.float64, device="cuda")
        want = fn(None).clone()
        g = _capture(lambda: fn(out))
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(_bits(out), _bits(want))


def test_sort_replay():
    """32-bit keys with HB_ASYNC never wait on the host, so the sort captures
    too; the replay sorts the same input to the same bits (stable payload)."""
    import torch

    n = 1_000_003
    src = torch.randint(0, 1 << 20, (n,), dtype=torch.int32, device="cuda")
    keys = src.clone()
    vals = torch.arange(n, dtype=torch.int32, device="cuda")

    def step():
        keys.copy_(src)
        vals.copy_(torch.arange(n, dtype=torch.int32, device="cuda"))
        gpu_sort(keys, vals, asynchronous=True)

    step()
    torch.cuda.synchronize()
    want_k, want_v = keys.clone(), vals.clone()
    g = _capture(step)
    keys.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(keys, want_k) and torch.equal(vals, want_v)
    assert torch.equal(want_k, torch.sort(src, stable=True).values)
