#!/bin/bash
# Per-policy replay times on C4 (serial attribution).
mkdir -p gpurun_out
for p in lru lfu belady ml; do
  timeout 900 python bench.py --policies $p --no-cpu-baseline --steps 2 --e2e-steps 1 > gpurun_out/bench_pol_$p.json 2> gpurun_out/bench_pol_$p.err
  python - bench_pol_$p <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['ms_per_step'], d['stages']['ms_serial_attribution'])
PY
done
