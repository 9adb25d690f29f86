#!/bin/bash
# K3-TC variants: launch-list durations (512 traces) and alternating C4 benches.
mkdir -p gpurun_out
B="python bench.py --traces 512 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
for G in 1 3 2; do
  MCB_K3_GROUPS=$G timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_score_tc --csv --log-file gpurun_out/l_v$G.csv $B > /dev/null 2>&1
  echo "variant $G"; python tools/launch_table.py gpurun_out/l_v$G.csv | head -2
done
for r in 1 2; do for G in 1 3; do
MCB_K3_GROUPS=$G timeout 900 python bench.py --no-cpu-baseline --steps 4 --e2e-steps 1 > gpurun_out/bench_c4_v$G.json 2> gpurun_out/bench_c4_v$G.err
python - bench_c4_v$G <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['stages']['ms_per_step']['k3_scorer'], d['stages']['ms_serial_attribution']['k3_scorer'])
PY
done; done
