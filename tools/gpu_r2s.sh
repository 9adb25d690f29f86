#!/bin/bash
# DRAM traffic per step of K3 / K4 (roofline.traffic) on C4, C3, C2.
mkdir -p gpurun_out
for w in c4 c3 c2; do
  timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --print-units base --csv --log-file gpurun_out/traffic_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/traffic_$w.log 2>&1
  python tools/traffic_json.py gpurun_out/traffic_$w.csv $w > gpurun_out/r2_${w}_traffic.json
  python -c "import json;d=json.load(open('gpurun_out/r2_${w}_traffic.json'));print('$w',d['k3'],d['k4'],d['k3_ms'],d['k4_ms'],d['calls_under_ncu'])"
done
