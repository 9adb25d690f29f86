#!/bin/bash
# C3 kernel split (launch list of one bench step, ML only and non-ML only).
mkdir -p gpurun_out
for p in ml lru,lfu,belady; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c3_$p.csv python bench.py --workload c3 --policies $p --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
echo "== $p"; python tools/launch_table.py gpurun_out/l_c3_$p.csv | grep -v "at::" | head -8
done
