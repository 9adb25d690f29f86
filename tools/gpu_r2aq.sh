#!/bin/bash
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for w in c3 c2 c1 c4; do
timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 5 --e2e-steps 2 > gpurun_out/b_$w.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/b_$w.json').read().strip().splitlines()[-1]); print('$w', f\"{d['value']:.3e}\", round(d['ms_per_step'],2), f\"{d['e2e']['value']:.3e}\", {k: round(v,2) for k,v in d['stages']['ms_serial_attribution'].items()})"
done
