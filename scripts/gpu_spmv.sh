mkdir -p gpurun_out
timeout 900 python -m pytest -x -q > gpurun_out/t_spmv.txt 2>&1
tail -5 gpurun_out/t_spmv.txt
timeout 600 python bench.py --workload spmv --no-cpu --e2e-steps 1 --e2e-share gpu > gpurun_out/bench_spmv.json 2> gpurun_out/bench_spmv.err
python - <<'P'
import json
d = json.load(open("gpurun_out/bench_spmv.json"))
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["parity"])
P
tail -5 gpurun_out/bench_spmv.err
