# e2e legs with the measured host+GPU split vs all-on-GPU (bench.py --e2e-share)
for w in ${WLS:-hist spmv conv bilat}; do
  for sh in calibrated gpu; do
    python bench.py --workload $w --steps 5 --no-cpu --e2e-steps 3 --e2e-share $sh | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$w', '$sh', round(e['value'],3), e['unit'], 'share', e.get('share'), 'h2d', e['h2d_bytes_per_step'], 'parity', d['parity'])"
  done
done
