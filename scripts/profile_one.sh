# ncu --set full capture of one workload's dominant kernel + its launch list:  bash scripts/profile_one.sh <workload> <kernel-regex>
w=$1; k=$2
mkdir -p gpurun_out/prof
ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/prof/$w -f \
    python bench.py --workload $w --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --e2e-share gpu > gpurun_out/prof/$w.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/prof/${w}_launches.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --e2e-share gpu > /dev/null 2>&1
