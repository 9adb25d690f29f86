#!/bin/bash
# A/B of the K4-wide kernel (HEAD in gpurun_old vs working tree): C4 replay stages, twice each.
L=paper_2601_17063_b200/lib/libmcb.so
cp $L /tmp/libmcb_new.so
for r in 1 2; do for v in new old; do
  if [ $v = old ]; then cp gpurun_old/libmcb_old.so $L; else cp /tmp/libmcb_new.so $L; fi
  timeout 900 python bench.py --no-cpu-baseline --steps 4 --e2e-steps 1 > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); a=d['stages']['ms_serial_attribution']; print('$v', round(d['ms_per_step'],1), round(a['k4_replay_non_ml'],2), round(a['k4_replay_ml'],2))"
done; done
cp /tmp/libmcb_new.so $L
