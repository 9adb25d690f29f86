#!/bin/bash
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log || exit 1
for ps in 2 3; do for w in c3 c1; do
MCB_SEG_PASSES=$ps timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/b.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$w passes $ps', f\"{d['value']:.3e}\", round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages']['ms_serial_attribution'].items()})"
done; done
