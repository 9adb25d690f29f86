#!/bin/bash
# C3 speculation passes / segment length sweep (ML and all policies).
mkdir -p gpurun_out
for cfg in "0 0" "3 0" "4 0" "3 512" "4 1024"; do
  set -- $cfg
  MCB_SEG_PASSES=$1 MCB_SEG_EV=$2 timeout 900 python bench.py --workload c3 --no-cpu-baseline --steps 3 --e2e-steps 1 > gpurun_out/sw.json 2> gpurun_out/sw.err
  python - "$cfg" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value']/1e9,2), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stages']['ms_serial_attribution'].items()}, d['segmented_replay'])
PY
done
