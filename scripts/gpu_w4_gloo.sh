#!/bin/bash
# Functional run of the whole bench as 4 gloo ranks sharing one GPU (world-4 exchange paths with the
# CUDA kernels; timings are not NCCL numbers).
mkdir -p gpurun_out/w4
HB_BENCH_BACKEND=gloo timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
   --master-port 29612 bench.py --gpus 4 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/w4/bench_w4.json 2> gpurun_out/w4/bench_w4.err
tail -5 gpurun_out/w4/bench_w4.err; head -c 2500 gpurun_out/w4/bench_w4.json
