#!/bin/bash
# float64 re-score: prefix occurrence masks by shared-memory atomics instead of a 32-ballot transpose
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-python-reference --e2e-steps 2 > gpurun_out/pol.json 2>/dev/null
python - <<'PY'
import json,sys
d=json.loads(open('gpurun_out/pol.json').read().strip().splitlines()[-1])
print(f"{d['value']:.3e}", round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages']['ms_serial_attribution'].items()}, d.get('parity',{}).get('equal'), d['roofline'].get('rescored_events_per_step'))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_rescore -c 3 --csv python bench.py --traces 1024 --steps 1 --warmup 1 --no-cpu-baseline --no-python-reference --e2e-steps 1 2>/dev/null | grep k_rescore | tail -3
