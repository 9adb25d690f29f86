#!/bin/bash
# K3-TC groups / weight-ring depth: 3 groups x 2 stages vs 2 groups x 6 stages (E = 64).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_score_tc_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for G in 3 2; do
MCB_K3_GROUPS=$G timeout 900 python bench.py --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_c4_g$G.json 2> gpurun_out/bench_c4_g$G.err
python - bench_c4_g$G <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['stages']['ms_serial_attribution'])
PY
done
