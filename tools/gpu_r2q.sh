#!/bin/bash
# Experiment: k_score_tc duration with and without weight loads (launch list, 512 traces).
mkdir -p gpurun_out
B="python bench.py --traces 512 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
for x in 0 1; do
  if [ $x = 1 ]; then export MCB_K3_SPIN=1; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_score_tc --csv --log-file gpurun_out/l_now$x.csv $B > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/l_now$x.csv | head -3
done
