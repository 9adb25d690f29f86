#!/bin/bash
# K3-TC iteration: tests, launch list + ncu of the scorer on C4 (256 traces), full C4 bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_score_tc_gpu.py -x -q -s > gpurun_out/tc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc_tests.log
tail -14 gpurun_out/tc_tests.log
grep -q "passed" gpurun_out/tc_tests.log && ! grep -q "failed\|error" gpurun_out/tc_tests.log || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4s.csv python bench.py --traces 256 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_c4s.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_score_tc|k_rescore' -c 2 -o gpurun_out/k3tc_c4 python bench.py --traces 256 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_k3tc.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['stages']['ms_serial_attribution'], d['e2e']['value'])
PY
