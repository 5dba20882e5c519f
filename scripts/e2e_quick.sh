#!/bin/bash
# e2e legs of the given workloads (no CPU baseline): bash scripts/e2e_quick.sh bilat conv sort lr
for w in "$@"; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); w=d if 'e2e' in d and 'workloads' not in d else d
e=w['e2e']; print('$w', round(w['value'],1), w['unit'], 'e2e', round(e['value'],2), e['unit'], 'ms', round(e['ms_per_step'],2), 'share', (e.get('share') or {}).get('fraction_a'))"
done
