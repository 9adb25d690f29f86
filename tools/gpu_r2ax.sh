#!/bin/bash
# Per-rank work of C4 at 2 / 4 / 8 GPUs (2048 / 1024 / 512 traces) and knob variants at 512.
for n in 2048 1024 512; do
  timeout 600 python bench.py --traces $n --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stages']['ms_serial_attribution'].items()}, d['segmented_replay'])"
done
for cfg in "WIDE_MIN=1000000000" "SEG_EV=512" "SEG_EV=1024"; do
  env MCB_$cfg timeout 600 python bench.py --traces 512 --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('512 $cfg', round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stages']['ms_serial_attribution'].items()}, d['segmented_replay'])"
done
