#!/bin/bash
# Round-2 evidence: --set full captures of the changed dominant kernels + per-workload launch lists.
mkdir -p gpurun_out/prof
cap() {  # workload kernel-regex skip
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$2 -s ${3:-1} -c 1 -o gpurun_out/prof/$1 -f \
    python bench.py --workload $1 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --e2e-share gpu > gpurun_out/prof/$1.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof/${1}_launches.csv python bench.py --workload $1 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 \
    --e2e-share gpu > /dev/null 2>&1
}
cap spmv spmv_sell_kernel 1
cap lr lr_walk_log_kernel 1
cap hist hist_striped_kernel 1
cap sort onesweep_rfk_kernel 2
ls -la gpurun_out/prof
