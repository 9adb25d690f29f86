#!/bin/bash
# Piecewise host upload: GPU suite, C4 bench (e2e) with 8 pieces and with 1.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
for u in 8 1; do
MCB_UPLOAD_PIECES=$u timeout 900 python bench.py --no-cpu-baseline --steps 4 --e2e-steps 3 > gpurun_out/bench_c4_u$u.json 2> gpurun_out/bench_c4_u$u.err
python - bench_c4_u$u <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['e2e'])
PY
done
