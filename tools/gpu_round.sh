#!/bin/bash
# Round evidence: parity tests, smoke, bench lines (ours c2 default + reference arm + c1), the per-kernel
# launch list, and one full ncu capture of the top kernels (separate commands from the bench timing).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --workload c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_score_tile|k_seg_spec|k_seg_finish' -s 12 -c 6 -o gpurun_out/full_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_c2.log 2>&1
tail -2 gpurun_out/ncu_full_c2.log; tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
for f in bench_c2 bench_ref bench_c1; do echo "== $f"; tail -c 1500 gpurun_out/$f.json; done
