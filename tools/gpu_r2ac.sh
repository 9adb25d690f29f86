#!/bin/bash
# ML order rows: GPU suite, C4 ML replay with / without order rows.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
for o in 1 0; do
MCB_ML_ORDER=$o timeout 900 python bench.py --no-cpu-baseline --steps 4 --e2e-steps 2 > gpurun_out/bench_c4_o$o.json 2> gpurun_out/bench_c4_o$o.err
python - bench_c4_o$o <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['stages']['ms_serial_attribution'], d['e2e']['value'])
PY
done
