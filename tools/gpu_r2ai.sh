#!/bin/bash
for x in default 8 default; do
  if [ $x = 8 ]; then export MCB_UPLOAD_PIECES=8; else unset MCB_UPLOAD_PIECES; fi
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err
  python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$x', round(d['ms_per_step'],1), round(d['e2e']['ms_per_step'],1))"
done
