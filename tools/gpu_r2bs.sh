#!/bin/bash
# thread speculation ML: next event's rank row by cp.async: GPU suite, C3
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-python-reference --e2e-steps 2 > gpurun_out/pol.json 2>/dev/null
python - <<'PY'
import json,sys
d=json.loads(open('gpurun_out/pol.json').read().strip().splitlines()[-1])
print(f"{d['value']:.3e}", round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages']['ms_serial_attribution'].items()}, d.get('parity',{}).get('equal'))
PY
