#!/bin/bash
# C1 and C2 kernel split (launch lists of one bench step).
for w in c1 c2; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
echo "== $w"; python tools/launch_table.py gpurun_out/l_$w.csv | grep -v "at::\|refgen\|router\|ar1" | head -14
done
