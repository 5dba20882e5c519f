#!/bin/bash
# SpMV iteration: parity tests, bench line (SELL default), CSR-kernel A/B, ncu of both kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --workload spmv --no-cpu --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('spmv', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity'], d['e2e']['value'])"
cat > /tmp/ab.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_1303_2171_b200.datasets import device_gen_csr
from paper_1303_2171_b200.kernels_irregular import spmv_preprocess, gpu_spmv
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare
m = device_gen_csr(1_000_000, 1_000_000, 42, 1.6e-5)
p = spmv_preprocess(m, Platform.build(1.0, 3.0), WorkShare.manual(0.0))
x = torch.rand(1_000_000, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for meth in ("exact", "exact_csr", "exact", "exact_csr"):
    for _ in range(5): gpu_spmv(p.permuted, x, 0, 1_000_000, y=y, perm=p.perm, method=meth, asynchronous=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): gpu_spmv(p.permuted, x, 0, 1_000_000, y=y, perm=p.perm, method=meth, asynchronous=True)
    b.record(); torch.cuda.synchronize()
    print(meth, "%.2f us" % (a.elapsed_time(b) / 50 * 1e3))
PY
timeout 300 python /tmp/ab.py
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:spmv_ -c 8 --csv python /tmp/ab.py 2>/dev/null > gpurun_out/spmv_ncu.csv
python - <<'PY'
import csv, collections
lines=open('gpurun_out/spmv_ncu.csv').read().splitlines()
i=[k for k,l in enumerate(lines) if l.startswith('"ID"')][0]
rows=list(csv.reader(lines[i:])); h=rows[0]
ki,mi,vi=h.index('Kernel Name'),h.index('Metric Name'),h.index('Metric Value')
agg=collections.OrderedDict()
for r in rows[1:]: agg.setdefault((r[0],r[ki][:40]),{})[r[mi]]=r[vi]
for k,m in agg.items(): print(k, {a.split('__')[-1][:40]:b for a,b in m.items()})
PY
