#!/bin/bash
# K1 v2 (persistent, 256x256 tiles, 3 x 64 KB stages): router tests, timing on C1/C3/C2 shapes, ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_router_gpu.py tests/test_fullsize_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
for w in c1 c3 c2; do timeout 300 python tools/prof_k1.py --workload $w --tokens 65536 --reps 10; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_topk -c 1 -o gpurun_out/k1v2_c1 python tools/prof_k1.py --workload c1 --tokens 65536 --reps 1 > gpurun_out/ncu_k1v2.log 2>&1
tail -1 gpurun_out/ncu_k1v2.log
