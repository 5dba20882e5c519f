# Filter kernel variants (HB_BILAT_CFG / HB_CONV_CFG, see bilateral.cu / conv.cu launch_tile).
for c in ${CFGS:-0 1}; do
  for w in bilat conv; do
    HB_BILAT_CFG=$c HB_CONV_CFG=$c python bench.py --workload $w --steps 10 --no-cpu --e2e-steps 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w cfg', '$c', d['ms_per_step'], d['value'], d['roofline'].get('compute', {}).get('achieved_gflops'), d['parity'])"
  done
done
