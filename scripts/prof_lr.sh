#!/bin/bash
# List-ranking iteration: parity tests, bench line, per-kernel ncu times + DRAM bytes of one step.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_listrank.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --workload lr --no-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lr', d['value'], d['ms_per_step'], d['parity'], d['e2e']['value'])"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lr_ -c 12 --csv \
  python bench.py --workload lr --no-cpu --steps 1 --warmup 3 --e2e-steps 1 2>/dev/null > gpurun_out/lr_ncu.csv
python scripts/ncu_agg.py gpurun_out/lr_ncu.csv | head -14
