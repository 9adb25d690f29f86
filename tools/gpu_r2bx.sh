#!/bin/bash
# e2e: host upload pieces (MCB_UPLOAD_PIECES) on C4
mkdir -p gpurun_out
for n in 8 16 32; do
MCB_UPLOAD_PIECES=$n timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-python-reference --e2e-steps 5 > gpurun_out/pol.json 2>/dev/null
python - $n <<'PY'
import json,sys
d=json.loads(open('gpurun_out/pol.json').read().strip().splitlines()[-1])
print('pieces', sys.argv[1], f"{d['value']:.3e}", round(d['ms_per_step'],2), 'e2e', f"{d['e2e']['value']:.3e}", round(d['e2e']['ms_per_step'],2))
PY
done
