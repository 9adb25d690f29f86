#!/bin/bash
# One full ncu capture of kernel $1 on workload $2 (policies $3) -> gpurun_out/$4.ncu-rep
mkdir -p gpurun_out
K=$1; W=${2:-c2}; POL=${3:-lru,lfu,belady,ml}; OUT=${4:-prof}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${5:-2} -c 1 -o gpurun_out/$OUT python bench.py --workload $W --policies $POL --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/$OUT.log 2>&1
tail -3 gpurun_out/$OUT.log
