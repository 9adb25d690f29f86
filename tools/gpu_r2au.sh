#!/bin/bash
# E = 128 scorer variants (C1 / C5 shapes): tests, then K3 time per variant on C1 and a C5 slice.
timeout 900 python -m pytest tests/test_score_tc_gpu.py tests/test_fullsize_oracle_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for G in 3 1; do
  for w in c1; do
  MCB_K3_GROUPS=$G timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$w v$G', round(d['ms_per_step'],3), round(d['stages']['ms_serial_attribution']['k3_scorer'],3))"
  done
  MCB_K3_GROUPS=$G timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_score_tc --csv --log-file gpurun_out/l_c5_$G.csv python bench.py --workload c5 --traces 256 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
  echo "c5 slice v$G"; python tools/launch_table.py gpurun_out/l_c5_$G.csv | head -1
done
