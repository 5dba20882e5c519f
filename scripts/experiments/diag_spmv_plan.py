"""Diagnostics of the column-ordered rounds SpMV plan on the 1M config:
plan geometry, round-size distribution, kernel time (CUDA events)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1303_2171_b200.datasets import device_gen_csr
from paper_1303_2171_b200.kernels_irregular import gpu_spmv, spmv_plan, spmv_preprocess
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
m = device_gen_csr(rows, rows, 42, 1.6e-5 * 1e6 / rows)
prep = spmv_preprocess(m, Platform.build(1.0, 3.0), WorkShare.manual(0.0))
dm, perm = prep.permuted, prep.perm
x = torch.rand(rows, dtype=torch.float64, device="cuda")
y = torch.empty(rows, dtype=torch.float64, device="cuda")
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
t0.record()
plan = spmv_plan(dm, 0, rows)
t1.record()
torch.cuda.synchronize()
print(f"build {t0.elapsed_time(t1):.2f} ms: chunks {plan.chunks} ctas {plan.ctas} rows/cta {plan.rows_per_cta} "
      f"rounds {plan.rounds} ({plan.rounds / max(plan.ctas * plan.chunks, 1):.1f}/cta, nnz/1024/cta "
      f"{plan.nnz / 1024 / max(plan.ctas * plan.chunks, 1):.1f}) bytes {plan.nbytes}")
for method in ("exact", "exact_sell"):
    for _ in range(3):
        gpu_spmv(dm, x, 0, rows, y=y, perm=perm, method=method, asynchronous=True)
    t0.record()
    for _ in range(20):
        gpu_spmv(dm, x, 0, rows, y=y, perm=perm, method=method, asynchronous=True)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / 20
    print(f"{method:11s} {ms * 1e3:8.1f} us  {2 * dm.nnz / ms / 1e6:7.1f} GFLOP/s")
