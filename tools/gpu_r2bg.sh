#!/bin/bash
# ncu --set full of the C1 ML warp speculation pass (the ML replay is C1's critical path)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wseg_spec --launch-skip 2 -c 2 -o gpurun_out/c1_wspec python bench.py --workload c1 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c1.log 2>&1
tail -2 gpurun_out/ncu_c1.log
