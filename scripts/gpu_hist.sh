timeout 600 python -m pytest tests/test_gpu_hist.py tests/test_gpu_graphs.py tests/test_gpu_fuzz.py tests/test_gpu_acceptance.py tests/test_capi.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -2
timeout 300 python scripts/prof_hist_sizes.py
timeout 300 python bench.py --workload hist --no-cpu --e2e-steps 2 > gpurun_out/hist.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/hist.json')); print(round(d['value'],1), d['unit'], round(d['ms_per_step']*1e3,1), 'us frac', round(d['roofline']['frac'],4), 'parity', d['parity'], d['e2e']['value'], d['e2e']['parity'])"
