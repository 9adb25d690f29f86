#!/bin/bash
# K4-wide LRU recency list + ML byte ranks, one launch per policy: GPU suite, C4 and C5 benches.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
timeout 900 python bench.py --no-cpu-baseline --steps 5 --e2e-steps 2 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 1200 python bench.py --workload c5 --no-cpu-baseline --steps 2 --e2e-steps 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for f in bench_c4 bench_c5; do python - $f <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['stages']['ms_serial_attribution'], d['e2e']['value'])
PY
done
