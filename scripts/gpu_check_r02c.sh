#!/bin/bash
# Re-entry check after the container was re-created: GPU suite + smoke + N=1 bench on the restored checkpoint.
O=gpurun_out/chk; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > $O/t_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; cp gpurun_out/bench_detail.json $O/bench_detail.json
cat $O/t_gpu.txt $O/smoke.txt; head -c 2500 $O/bench.json; echo
