#!/bin/bash
# K3-TC fp16x2: scorer tests, C4 bench (3 and 2 groups), ncu of the scorer.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_score_tc_gpu.py -x -q -s -p no:cacheprovider > gpurun_out/tc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc_tests.log
grep -v "^$" gpurun_out/tc_tests.log | tail -32
grep -q "passed" gpurun_out/tc_tests.log && ! grep -q "failed\|error" gpurun_out/tc_tests.log || exit 1
timeout 900 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
MCB_K3_GROUPS=2 timeout 900 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_c4_g2.json 2> gpurun_out/bench_c4_g2.err
for f in bench_c4 bench_c4_g2; do python - $f <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['stages']['ms_serial_attribution'], d['e2e']['value'], d['roofline']['frac'], d['rooflines']['k3_scorer'].get('rescored_events_per_step'))
PY
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_score_tc' -c 1 -o gpurun_out/k3tc16_c4 python bench.py --traces 512 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_k3tc.log 2>&1
tail -1 gpurun_out/ncu_k3tc.log
