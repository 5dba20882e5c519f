"""Device-side generators: HBM streams bit-identical to
the reference generators, including offset (k0) chunks for sharded runs."""

import numpy as np
import pytest

from oracle import datasets as ods
from paper_1303_2171_b200 import datasets as d

pytestmark = pytest.mark.gpu


def test_device_sort_hist_image_generators():
    n = 100_003
    keys = d.device_gen_sort_data(n, 42).cpu().numpy().view(np.uint32)
    assert np.array_equal(keys.astype(np.int64), d.gen_sort_data(n, 42))
    tail = d.device_gen_sort_data(1000, 42, k0=n - 1000).cpu().numpy().view(np.uint32)
    assert np.array_equal(tail, keys[-1000:])
    for bins in (256, 100, 1000):
        got = d.device_gen_hist_data(n, 7, bins).cpu().numpy()
        assert np.array_equal(got.astype(np.int64), d.gen_hist_data(n, 7, bins)), bins
    assert np.array_equal(d.device_gen_image(77, 3).cpu().numpy(), d.gen_image(77, 3).pixels)
    assert np.array_equal(d.gen_image(77, 3).pixels, ods.image(77, 3))


def test_device_gen_list_matches_reference_generator():
    succ, head = d.device_gen_list(50_000, 11)
    want = d.gen_list(50_000, 11)
    assert head == want.head and np.array_equal(succ.cpu().numpy().astype(np.int64), want.succ)


def test_worker_threads_inherit_the_callers_device():
    """run_workshared's side threads must run on the rank's GPU (a new
    host thread starts on device 0): the wrapper carries the device over."""
    import threading

    import torch

    from paper_1303_2171_b200.gpu import inherit_device

    last = torch.cuda.device_count() - 1
    torch.cuda.set_device(last)
    seen = []
    t = threading.Thread(target=inherit_device(lambda: seen.append(torch.cuda.current_device())))
    t.start()
    t.join()
    torch.cuda.set_device(0)
    assert seen == [last]


@pytest.mark.parametrize("rows,cols,seed,density", [
    (100_000, 100_000, 42, 1.6e-4),   # ~16 nnz/row, like the 1M config
    (20_000, 1_000_000, 7, 1.6e-5),
    (5_000, 50, 3, 0.2),              # dense-ish rows (up to 19 of 50 columns)
    (3_000, 10, 5, 0.5),              # 10 columns: rows that need the retry loop
    (1, 1, 9, 1.0),
])
def test_device_gen_csr_matches_reference_generator(rows, cols, seed, density):
    """hb_gen_csr == csr_arrays (itself pinned to the reference's gen_csr by
    the golden fixtures), including rows that take extra stream draws."""
    ptr, col, val = d.csr_arrays(rows, cols, seed, density)
    for idx in (np.int32, np.int64):
        m = d.device_gen_csr(rows, cols, seed, density, idx)
        assert np.array_equal(m.row_ptr.cpu().numpy().astype(np.int64), ptr)
        assert np.array_equal(m.col_idx.cpu().numpy().astype(np.int64), col)
        assert np.array_equal(m.values.cpu().numpy().view(np.uint64), val.view(np.uint64))


def test_device_gen_csr_at_config_size():
    m = d.device_gen_csr(1_000_000, 1_000_000, 42, 1.6e-5)
    assert m.nnz == 15_989_277  # the reference's nnz at the SpMV config
