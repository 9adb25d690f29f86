#!/bin/bash
# K4-wide profile on C4 (1024 traces: both the non-ML and the ML launch take
# the thread-per-instance kernel), and racecheck of the fixed fp64 scorer.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_replay_wide -c 2 -o gpurun_out/k4w_c4 python bench.py --traces 1024 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_k4w.log 2>&1
tail -2 gpurun_out/ncu_k4w.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_parity_gpu.py::test_scorer_ranks_match_scores tests/test_parity_gpu.py::test_small_cases -q -x -p no:cacheprovider > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.log
tail -3 gpurun_out/sanitize_racecheck.log
