#!/bin/bash
# Round-2 profiling pack: C4 launch list (512 traces), ncu --set full of the
# K3-TC scorer, the K4-wide replay, K2 next-use, and K1 on the C1/C3 shapes.
mkdir -p gpurun_out
B="python bench.py --traces 512 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu_launch_c4.log 2>&1
python tools/launch_table.py gpurun_out/launches_c4.csv | head -30
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_score_tc|k_rescore|k_snap|k_tile_summary|k_next_use|k_replay_wide' -c 8 -o gpurun_out/c4_full $B > gpurun_out/ncu_c4_full.log 2>&1
tail -2 gpurun_out/ncu_c4_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_topk -c 1 -o gpurun_out/k1_c3 python tools/prof_k1.py --workload c3 --tokens 65536 --reps 1 > gpurun_out/ncu_k1_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_topk -c 1 -o gpurun_out/k1_c1 python tools/prof_k1.py --workload c1 --tokens 65536 --reps 1 > gpurun_out/ncu_k1_c1.log 2>&1
tail -2 gpurun_out/ncu_k1_c1.log
