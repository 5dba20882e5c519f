#!/bin/bash
# Round-2 GPU pass: sharded/gen_csr tests, N=1 bench, 2-rank gloo functional bench, reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_datasets.py -x -q 2>&1 | tail -30 > gpurun_out/t_new.txt
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
HB_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
   --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/bench_w2.json 2> gpurun_out/bench_w2.err
cp gpurun_out/bench_detail.json gpurun_out/bench_w2_detail.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
cat gpurun_out/t_new.txt; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err; cat gpurun_out/bench_w2.json; tail -20 gpurun_out/bench_w2.err; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
