#!/bin/bash
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_snap_scan|k_tile_summary' --csv --log-file gpurun_out/l_snap.csv python bench.py --traces 512 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/l_snap.csv | head -3
