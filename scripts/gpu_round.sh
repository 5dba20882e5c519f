#!/bin/bash
# One gpurun round-trip: build check, GPU tests, smoke, bench, ncu launch list + full capture of the top kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt
python -m pytest tests -x -q -m gpu 2>&1 | tail -25 > gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ -n "${NCU:-}" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu ${NCU_ARGS:-} > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-hist} -s 3 -c 1 \
      -o gpurun_out/prof -f python bench.py --steps 3 --warmup 3 --no-cpu ${NCU_ARGS:-} > gpurun_out/ncu_full.log 2>&1
fi
tail -5 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt | tail -3; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
