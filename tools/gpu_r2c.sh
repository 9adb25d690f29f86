#!/bin/bash
# K3-TC profile on C4 (256 traces): launch list + full ncu of the TC scorer and the re-score.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4s.csv python bench.py --traces 256 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_c4s.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_score_tc|k_rescore' -c 2 -o gpurun_out/k3tc_c4 python bench.py --traces 256 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_k3tc.log 2>&1
tail -3 gpurun_out/ncu_k3tc.log
