#!/bin/bash
# Quick GPU iteration: parity tests + bench lines (no ncu).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for w in c2 c1; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  python - $w <<'PY'
import json,sys
w=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/bench_{w}.json").read().strip().splitlines()[-1])
    print(w, "value %.3e" % d["value"], "ms %.3f" % d["ms_per_step"], {k:(round(v,3) if isinstance(v,float) else '') for k,v in d["config"]["stage_ms_per_step"].items() if k!="note"}, "e2e %.3e" % d["e2e"]["value"])
except Exception as e:
    print(w, "FAILED", e); print(open(f"gpurun_out/bench_{w}.err").read()[-3000:])
PY
done
