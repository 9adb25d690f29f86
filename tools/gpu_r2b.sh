#!/bin/bash
# K3-TC first light: the tensor-core scorer's tests, then the C4 bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_score_tc_gpu.py -x -q -s > gpurun_out/tc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc_tests.log
tail -30 gpurun_out/tc_tests.log
if grep -q "passed" gpurun_out/tc_tests.log && ! grep -q "failed\|error" gpurun_out/tc_tests.log; then
  timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
  timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
  tail -c 2500 gpurun_out/bench_c4.json
fi
