#!/bin/bash
# GPU pass: full GPU suite, smoke, N=1 bench, reference arm.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -25 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -8 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/smoke.txt; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
