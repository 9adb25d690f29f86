#!/bin/bash
# warp segmented replay with packed keys and sequential cursors: tests + C1 / C3
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for w in c1 c3; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c1s.json 2>/dev/null
python - $w <<'PY'
import json,sys
d=json.loads(open('gpurun_out/c1s.json').read().strip().splitlines()[-1])
print(sys.argv[1], f"{d['value']:.3e}", round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages']['ms_serial_attribution'].items()}, d['segmented_replay'], d.get('parity'))
PY
done
