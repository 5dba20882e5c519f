#!/bin/bash
# ncu --set full capture of each workload's dominant kernel + the launch list of one bench step.
mkdir -p gpurun_out/prof
for spec in "hist:hist_striped" "spmv:spmv_lpr" "sort:onesweep_rfk" "bilat:bilateral_tma" "conv:conv_rows" "lr:lr_walk_kernel"; do
  w=${spec%%:*}; k=${spec##*:}
  ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/prof/$w -f \
      python bench.py --workload $w --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/prof/$w.log 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/prof/${w}_launches.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
done
ls -la gpurun_out/prof
