#!/bin/bash
# K1 ncu captures (fixed launch skip), C5 one-step bench, then the sanitizer pass.
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_topk -s 1 -c 1 -o gpurun_out/k1_c3 python tools/prof_k1.py --workload c3 --tokens 65536 --reps 1 > gpurun_out/ncu_k1_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_topk -s 1 -c 1 -o gpurun_out/k1_c1 python tools/prof_k1.py --workload c1 --tokens 65536 --reps 1 > gpurun_out/ncu_k1_c1.log 2>&1
tail -2 gpurun_out/ncu_k1_c3.log
timeout 1500 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -c 1200 gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
bash tools/gpu_sanitize.sh
