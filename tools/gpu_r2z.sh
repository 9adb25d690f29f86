#!/bin/bash
# ncu of the C3 ML finish walk (k_wseg_finish) with source lines.
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_wseg_finish -c 1 -o gpurun_out/c3_fin python bench.py --workload c3 --policies ml --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c3_fin.log 2>&1
tail -1 gpurun_out/ncu_c3_fin.log
