# SpMV variant sweep: HB_SPMV_CFG selects the kernel (spmv.cu launch_spmv); prints ms/step, GFLOP/s, HBM frac, parity.
for c in ${CFGS:-0 1}; do HB_SPMV_CFG=$c python bench.py --workload spmv --steps 20 --no-cpu --e2e-steps 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg', '$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['parity'])"; done
for c in ${NCU_CFGS:-}; do
  HB_SPMV_CFG=$c ncu --metrics gpu__time_duration.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sectors_lookup_miss.sum --clock-control none -k regex:spmv_ -s 2 -c 1 python bench.py --workload spmv --steps 2 --warmup 3 --no-cpu --e2e-steps 1 2>&1 | grep -E "spmv_|gpu__|l1tex|dram__|warps" | sed "s/^/cfg $c /"
done
