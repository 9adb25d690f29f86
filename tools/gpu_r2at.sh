#!/bin/bash
# C1 warp speculation sweep: passes / segment length / warm-up.
for cfg in "0 0 0" "1 0 0" "1 256 128" "1 512 256" "2 512 256" "2 256 64" "1 1024 512" "2 128 64"; do
  set -- $cfg
  MCB_SEG_PASSES=$1 MCB_SEG_EV=$2 MCB_SEG_NW=$3 timeout 600 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c1s.json 2>/dev/null
  python - "$cfg" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/c1s.json').read().strip().splitlines()[-1])
print(sys.argv[1], f"{d['value']:.3e}", round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages']['ms_serial_attribution'].items()}, d['segmented_replay']['fixup_events'], d['segmented_replay']['segments'])
PY
done
