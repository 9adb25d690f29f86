#!/bin/bash
# Round-2 numbers on every workload + C4 launch list (full size).
mkdir -p gpurun_out
for w in c1 c2 c3; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 5 --e2e-steps 2 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  python - $w <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/bench_{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['stages']['ms_serial_attribution'], d['e2e']['value'], d.get('generator',{}) and d['generator'].get('frac_of_bf16_peak'))
PY
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_full.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_c4_full.log 2>&1
python tools/launch_table.py gpurun_out/launches_c4_full.csv | head -20
