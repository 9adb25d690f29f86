#!/bin/bash
# Experiment: K3-TC without weight loads (timing only), and a 2-rank bench on one GPU.
mkdir -p gpurun_out
for x in 0 1; do
  if [ $x = 1 ]; then export MCB_K3_EXP_NOW=1; fi
  timeout 900 python bench.py --no-cpu-baseline --steps 3 --e2e-steps 1 > gpurun_out/bench_now$x.json 2> gpurun_out/bench_now$x.err
  python - bench_now$x <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['stages']['ms_serial_attribution'])
PY
done
unset MCB_K3_EXP_NOW
timeout 900 python bench.py --gpus 2 --no-cpu-baseline --steps 3 --e2e-steps 1 > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo "2rank rc=$?"
tail -c 600 gpurun_out/bench_2rank.json; tail -3 gpurun_out/bench_2rank.err
