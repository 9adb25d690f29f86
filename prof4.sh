B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --policies lru"
MCB_SOLO_MIN=100000000 ncu --set full --clock-control none --import-source on -k regex:'k_replay' -s 3 -c 1 -o gpurun_out/prof_lru_warp $B > gpurun_out/p4.log 2>&1
MCB_SOLO_MIN=0 ncu --set full --clock-control none --import-source on -k regex:'k_replay' -s 3 -c 1 -o gpurun_out/prof_lru_solo $B >> gpurun_out/p4.log 2>&1
tail -2 gpurun_out/p4.log
