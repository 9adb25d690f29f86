#!/bin/bash
# Round 2, first GPU pass: GPU tests, the C4 headline + reference arm, and
# the K1 / K2 ncu captures the round-1 verdict asked for.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference --steps 3 > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref_c4.err
for w in c3 c1 c2; do timeout 300 python tools/prof_k1.py --workload $w --tokens 65536 > gpurun_out/k1_$w.json 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_topk -s 2 -c 1 -o gpurun_out/k1_c3 python tools/prof_k1.py --workload c3 --tokens 65536 --reps 1 > gpurun_out/ncu_k1_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_topk -s 2 -c 1 -o gpurun_out/k1_c1 python tools/prof_k1.py --workload c1 --tokens 65536 --reps 1 > gpurun_out/ncu_k1_c1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_next_use -c 2 -o gpurun_out/k2_c4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_k2_c4.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -2
for f in bench_c4 bench_ref_c4 k1_c3 k1_c1 k1_c2; do echo "== $f"; tail -c 600 gpurun_out/$f.json; done
