#!/bin/bash
# Per-kernel launch list (cold, serialized) of one bench step.
mkdir -p gpurun_out
W=${1:-c2}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_$W.log 2>&1
python tools/launch_table.py gpurun_out/launches_$W.csv
