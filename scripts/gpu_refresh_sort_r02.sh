#!/bin/bash
# Refresh after the sort look-back changes: N=1 bench line, largest shapes, and the sort's ncu evidence.
O=gpurun_out/final; mkdir -p $O/prof
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; cp gpurun_out/bench_detail.json $O/bench_detail.json
timeout 1200 python bench.py --shape largest --scaling strong --steps 5 --no-cpu > $O/bench_largest.json 2> $O/bench_largest.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:onesweep_rfk_kernel -s 11 -c 1 -o $O/prof/sort -f \
  python bench.py --workload sort --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --e2e-share gpu > $O/prof/sort.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/prof/sort_launches.csv python bench.py --workload sort --steps 1 --warmup 3 --no-cpu --e2e-steps 1 \
  --e2e-share gpu > /dev/null 2>&1
head -c 2600 $O/bench.json
