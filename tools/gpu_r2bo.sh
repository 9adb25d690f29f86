#!/bin/bash
# C4 launch list of the current kernels + ncu --set full of K4-wide (both launches) and the float64 re-score
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-python-reference --e2e-steps 1 > gpurun_out/ncu_launch_c4.log 2>&1
python tools/launch_table.py gpurun_out/launches_c4.csv > gpurun_out/launches_c4_table.txt 2>&1; head -30 gpurun_out/launches_c4_table.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_replay_wide|k_rescore' -s 3 -c 3 -o gpurun_out/c4_tail python bench.py --traces 1024 --steps 1 --warmup 1 --no-cpu-baseline --no-python-reference --e2e-steps 1 > gpurun_out/ncu_tail.log 2>&1
tail -2 gpurun_out/ncu_tail.log
