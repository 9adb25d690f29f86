#!/bin/bash
for cfg in "WIDE_MIN=16384" "WIDE_MIN=8192" "WIDE_MIN=2048"; do
 for n in 512 256; do
  env MCB_$cfg timeout 600 python bench.py --traces $n --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$n $cfg', round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stages']['ms_serial_attribution'].items()})"
 done
done
