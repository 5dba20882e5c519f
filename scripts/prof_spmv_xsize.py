"""SpMV time at 2^24 rows, ~16 nnz/row, as the x vector shrinks (cols = rows / d): how much of the
largest shape's loss is x outgrowing L2 (the potential of column blocking).  gpu_spmv on the
nnz-sorted device matrix, CUDA events, mean of 10 calls."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1303_2171_b200.datasets import device_gen_csr
from paper_1303_2171_b200.kernels_irregular import gpu_spmv, spmv_preprocess
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

rows = 1 << 24
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for d in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 16]:
    cols = rows // d
    m = device_gen_csr(rows, cols, 42, 16.0 / cols)
    nnz = m.nnz
    prep = spmv_preprocess(m, Platform.build(1.0, 3.0), WorkShare.manual(0.0))
    del m
    x = torch.rand(cols, dtype=torch.float64, device="cuda")
    y = torch.empty(rows, dtype=torch.float64, device="cuda")
    for _ in range(3):
        gpu_spmv(prep.permuted, x, 0, rows, y=y, perm=prep.perm, asynchronous=True)
    e0.record()
    for _ in range(10):
        gpu_spmv(prep.permuted, x, 0, rows, y=y, perm=prep.perm, asynchronous=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cols = rows/{d:<3d} (x {cols * 8 / 1e6:6.1f} MB): nnz {nnz}  {ms:.3f} ms  {2 * nnz / ms / 1e6:.1f} GFLOP/s", flush=True)
    del prep, x, y
    torch.cuda.empty_cache()
