#!/bin/bash
# K3-TC half-jobs: scorer tests, then A/B (HEAD in gpurun_old vs working tree): launch list + C4 bench.
timeout 900 python -m pytest tests/test_score_tc_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
B="python bench.py --traces 512 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
L=paper_2601_17063_b200/lib/libmcb.so
cp $L /tmp/libmcb_new.so
for v in new old new; do
  if [ $v = old ]; then cp gpurun_old/libmcb_old.so $L; else cp /tmp/libmcb_new.so $L; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_score_tc --csv --log-file gpurun_out/l_$v.csv $B > /dev/null 2>&1
  echo "$v"; python tools/launch_table.py gpurun_out/l_$v.csv | head -1
done
cp /tmp/libmcb_new.so $L
timeout 900 python bench.py --no-cpu-baseline --steps 4 --e2e-steps 1 > gpurun_out/ab.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],1), d['stages']['ms_serial_attribution'])"
