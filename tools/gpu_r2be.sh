#!/bin/bash
# C1: segmented (default) vs one warp per instance (MCB_SEG_EV=-1)
for ev in 0 -1; do
  MCB_SEG_EV=$ev timeout 600 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c1s.json 2>/dev/null
  python - "$ev" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/c1s.json').read().strip().splitlines()[-1])
print(sys.argv[1], f"{d['value']:.3e}", round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages']['ms_serial_attribution'].items()}, d['segmented_replay'])
PY
done
