#!/bin/bash
timeout 600 python tools/var_probe.py 25 2>&1 | awk '{print $1, $3}' | tr '\n' ' '; echo
timeout 600 python tools/e2e_ab.py
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --steps 8 --e2e-steps 8 > gpurun_out/b.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],1), d['e2e']['ms_per_step'], d['e2e']['value'], d['value'])"
done
