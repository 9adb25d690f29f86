#!/bin/bash
# K3-TC epilogue diet + K4-wide key scan: GPU suite, C4 bench, ncu of both kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_score_tc_gpu.py -x -q -s -p no:cacheprovider > gpurun_out/tc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc_tests.log
grep "max normwise\|passed\|failed\|rc=" gpurun_out/tc_tests.log
grep -q "passed" gpurun_out/tc_tests.log && ! grep -q "failed\|error" gpurun_out/tc_tests.log || exit 1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python - bench_c4 <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['stages']['ms_serial_attribution'], d['e2e']['value'], d['roofline']['frac'])
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_score_tc|k_replay_wide' -c 3 -o gpurun_out/c4_r2k python bench.py --traces 2048 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_r2k.log 2>&1
tail -1 gpurun_out/ncu_r2k.log
