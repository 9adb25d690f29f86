#!/bin/bash
# Session re-entry check of HEAD: GPU suite, smoke, C4 headline + reference arm, C1 / C3 lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for w in c1 c3; do timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
for f in bench_c4 bench_ref bench_c1 bench_c3; do echo "== $f"; python - gpurun_out/$f.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), d.get('parity'), (d.get('roofline') or {}).get('frac'), d.get('clocks'))
except Exception as e: print('ERR', e)
PY
done
