#!/bin/bash
for G in 3 1 3 1; do
  MCB_K3_GROUPS=$G timeout 600 python bench.py --workload c2 --no-cpu-baseline --steps 10 --e2e-steps 1 > gpurun_out/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('c2 v$G', round(d['ms_per_step'],3), round(d['stages']['ms_serial_attribution']['k3_scorer'],3))"
done
