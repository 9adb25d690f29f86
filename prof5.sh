B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --policies ml"
ncu --set full --clock-control none --import-source on -k regex:'k_score_tile' -s 3 -c 1 -o gpurun_out/prof_score_c2 $B > gpurun_out/p5.log 2>&1
tail -1 gpurun_out/p5.log
