#!/bin/bash
# K4-wide on C4: per-policy stage times, the 512-trace (8-GPU per-rank) step, ncu source view of both launches
mkdir -p gpurun_out
for p in lru lfu belady ml lru,lfu,belady; do
timeout 600 python bench.py --policies $p --steps 5 --warmup 3 --no-cpu-baseline --no-python-reference --e2e-steps 1 > gpurun_out/pol.json 2>/dev/null
python - $p <<'PY'
import json,sys
d=json.loads(open('gpurun_out/pol.json').read().strip().splitlines()[-1])
print(sys.argv[1], round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages']['ms_serial_attribution'].items()})
PY
done
for t in 512 1024; do
timeout 600 python bench.py --traces $t --steps 5 --warmup 3 --no-cpu-baseline --no-python-reference --e2e-steps 1 > gpurun_out/pol.json 2>/dev/null
python - $t <<'PY'
import json,sys
d=json.loads(open('gpurun_out/pol.json').read().strip().splitlines()[-1])
print('traces', sys.argv[1], round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages']['ms_serial_attribution'].items()}, {k: round(v,2) for k,v in d['stages']['ms_per_step'].items()})
PY
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_replay_wide -s 2 -c 2 -o gpurun_out/wide_c4 python bench.py --traces 1024 --steps 1 --warmup 1 --no-cpu-baseline --no-python-reference --e2e-steps 1 > gpurun_out/ncu_wide.log 2>&1
tail -2 gpurun_out/ncu_wide.log
