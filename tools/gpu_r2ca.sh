#!/bin/bash
# ML replay with a third speculation pass under thread speculation (C3): GPU suite, C3, C4 unchanged
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for a in "--workload c3" "--workload c3 --steps 10"; do
timeout 600 python bench.py $a --warmup 3 --no-python-reference --e2e-steps 2 > gpurun_out/pol.json 2>/dev/null
python - "$a" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/pol.json').read().strip().splitlines()[-1])
print(sys.argv[1], f"{d['value']:.3e}", round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages']['ms_serial_attribution'].items()}, d['segmented_replay'], (d.get('parity') or {}).get('equal'))
PY
done
