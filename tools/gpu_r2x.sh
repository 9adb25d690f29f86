#!/bin/bash
# tspec word-wise scan + ML byte ranks: GPU suite, C3 and C4 benches.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
for w in c3 c4; do
timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 4 --e2e-steps 1 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
python - bench_$w <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['stages']['ms_serial_attribution'], d['segmented_replay'])
PY
done
