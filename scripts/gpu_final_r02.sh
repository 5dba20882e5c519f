#!/bin/bash
# Round-2 closing pass on one B200: full GPU suite + smoke, the N=1 bench line, the reference arm, the
# 2-rank gloo functional run, the largest shapes, and per-workload ncu evidence (launch lists + one
# --set full capture of each dominant kernel).  Everything lands in gpurun_out/final/.
O=gpurun_out/final; rm -rf $O; mkdir -p $O/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/t_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; cp gpurun_out/bench_detail.json $O/bench_detail.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
HB_BENCH_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
   --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 2 > $O/bench_w2.json 2> $O/bench_w2.err
timeout 1200 python bench.py --shape largest --scaling strong --steps 5 --no-cpu > $O/bench_largest.json 2> $O/bench_largest.err
cap() {  # workload kernel-regex skip
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$2 -s ${3:-1} -c 1 -o $O/prof/$1 -f \
    python bench.py --workload $1 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --e2e-share gpu > $O/prof/$1.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/prof/${1}_launches.csv python bench.py --workload $1 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 \
    --e2e-share gpu > /dev/null 2>&1
}
cap hist hist_striped_kernel 1
cap spmv spmv_sell_kernel 1
cap sort onesweep_rfk_kernel 11  # skip the 10 launches of the device self-test (2^20 keys): capture the first packed 2^28 pass
cap lr lr_walk_log_kernel 1
cap bilat bilateral_tma_kernel 1
cap conv conv_rows_kernel 1
cat $O/t_gpu.txt $O/smoke.txt; head -c 600 $O/bench.json; echo; head -c 300 $O/bench_ref.json; echo; head -c 300 $O/bench_w2.json; echo
tail -3 $O/bench_w2.err; ls -la $O/prof
