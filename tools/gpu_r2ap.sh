#!/bin/bash
# C3 with 3 speculation passes: kernel split, ML only / non-ML only.
export MCB_SEG_PASSES=3
for p in ml lru,lfu,belady; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c3p3_$p.csv python bench.py --workload c3 --policies $p --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
echo "== $p"; python tools/launch_table.py gpurun_out/l_c3p3_$p.csv | grep -v "at::\|router\|ar1" | head -8
done
unset MCB_SEG_PASSES
for ps in 2 3; do
MCB_SEG_PASSES=$ps timeout 900 python bench.py --workload c3 --no-cpu-baseline --steps 4 --e2e-steps 1 > gpurun_out/c3p.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/c3p.json').read().strip().splitlines()[-1]); print('$ps', round(d['ms_per_step'],1), d['stages'])"
done
