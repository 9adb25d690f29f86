#!/bin/bash
# Round-2 final evidence: GPU suite, C4 bench + reference arm, C4 launch list, ncu --set full of the
# final K3-TC and K4-wide kernels (2,048 traces), racecheck / memcheck of the changed kernels.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_final.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_c4_final.csv | head -14
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_score_tc|k_replay_wide|k_snap_scan' -c 4 -o gpurun_out/c4_final python bench.py --traces 2048 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c4_final.log 2>&1
tail -1 gpurun_out/ncu_c4_final.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_score_tc_gpu.py -q -x -p no:cacheprovider -k "equal_float64_ranks" > gpurun_out/sanitize_racecheck_r2final.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck_r2final.log
tail -2 gpurun_out/sanitize_racecheck_r2final.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "small_cases" > gpurun_out/sanitize_memcheck_r2final.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck_r2final.log
tail -2 gpurun_out/sanitize_memcheck_r2final.log
