"""SpMV kernel time on the bench configs (1M rows and 2^24 rows, ~16 nnz/row,
nnz-sorted device matrix), CUDA events, mean of 50 calls, best of 3 — for A/B
runs of two library builds (HB200_LIB)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1303_2171_b200.datasets import device_gen_csr
from paper_1303_2171_b200.kernels_irregular import gpu_spmv, spmv_preprocess
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rows in [int(a) for a in sys.argv[1:]] or [1_000_000]:
    m = device_gen_csr(rows, rows, 42, 16.0 / rows)
    nnz = m.nnz
    prep = spmv_preprocess(m, Platform.build(1.0, 3.0), WorkShare.manual(0.0))
    del m
    x = torch.rand(rows, dtype=torch.float64, device="cuda")
    y = torch.empty(rows, dtype=torch.float64, device="cuda")
    best = 1e9
    for _ in range(3):
        for _ in range(5):
            gpu_spmv(prep.permuted, x, 0, rows, y=y, perm=prep.perm, asynchronous=True)
        e0.record()
        for _ in range(50):
            gpu_spmv(prep.permuted, x, 0, rows, y=y, perm=prep.perm, asynchronous=True)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 50)
    print(f"{os.environ.get('HB200_LIB', 'default'):40s} rows {rows:9d} nnz {nnz}: {best * 1e3:7.2f} us  "
          f"{2 * nnz / best / 1e6:6.1f} GFLOP/s", flush=True)
    del prep, x, y
    torch.cuda.empty_cache()
