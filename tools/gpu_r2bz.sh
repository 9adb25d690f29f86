#!/bin/bash
# C3: speculation passes of the segmented replay (MCB_SEG_PASSES) with the cheaper thread speculation
mkdir -p gpurun_out
for n in 0 2 3 4; do
MCB_SEG_PASSES=$n timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline --no-python-reference --e2e-steps 1 > gpurun_out/pol.json 2>/dev/null
python - $n <<'PY'
import json,sys
d=json.loads(open('gpurun_out/pol.json').read().strip().splitlines()[-1])
print('passes', sys.argv[1], f"{d['value']:.3e}", round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages']['ms_serial_attribution'].items()}, d['segmented_replay'])
PY
done
