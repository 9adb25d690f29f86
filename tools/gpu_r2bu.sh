#!/bin/bash
# C1 launch list (which replay kernels, how long)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --workload c1 --steps 1 --warmup 3 --no-cpu-baseline --no-python-reference --e2e-steps 1 > gpurun_out/ncu_launch_c1.log 2>&1
python tools/launch_table.py gpurun_out/launches_c1.csv > gpurun_out/launches_c1_table.txt 2>&1; head -25 gpurun_out/launches_c1_table.txt
