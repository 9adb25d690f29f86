#!/bin/bash
# K3-TC variant 1 (operands in TMEM, 2 groups, deep weight ring) vs 3 (smem operands, 3 groups).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_score_tc_gpu.py -x -q -s -p no:cacheprovider > gpurun_out/tc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc_tests.log
grep "groups\|normwise\|passed\|failed\|rc=\|Error" gpurun_out/tc_tests.log | head -30
grep -q "passed" gpurun_out/tc_tests.log && ! grep -q "failed\|error" gpurun_out/tc_tests.log || exit 1
for G in 1 3; do
MCB_K3_GROUPS=$G timeout 900 python bench.py --no-cpu-baseline --steps 3 --e2e-steps 1 > gpurun_out/bench_c4_v$G.json 2> gpurun_out/bench_c4_v$G.err
python - bench_c4_v$G <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['stages']['ms_serial_attribution'])
PY
done
