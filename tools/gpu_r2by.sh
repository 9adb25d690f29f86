#!/bin/bash
# K4-wide: resident count kept in a register instead of a popcount per miss
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for a in "--policies lru,lfu,belady" "--policies ml" ""; do
timeout 600 python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline --no-python-reference --e2e-steps 1 > gpurun_out/pol.json 2>/dev/null
python - "$a" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/pol.json').read().strip().splitlines()[-1])
print(sys.argv[1], f"{d['value']:.3e}", round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages']['ms_serial_attribution'].items()})
PY
done
