# list-ranking walk: chains per thread (HB_LR_LC; 1 = lr_walk_log_kernel, -1/2/3/4 = lr_walk_logm_kernel<LC>)
for lc in 1 -1 2 3 4; do
  HB_LR_LC=$lc timeout 300 python bench.py --workload lr --no-cpu --e2e-steps 1 --e2e-share gpu > gpurun_out/lr_lc$lc.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/lr_lc$lc.json')); print('LC=$lc', round(d['value'],1), d['unit'], round(d['ms_per_step'],3), 'ms parity', d['parity'])"
done
for lc in 2 3; do HB_LR_LC=$lc timeout 600 python -m pytest tests/test_gpu_listrank.py -x -q 2>&1 | tail -2; done
