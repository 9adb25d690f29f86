#!/bin/bash
# Final round-2 evidence: GPU suite, smoke, every workload's bench line + reference arm, C4 launch list,
# racecheck / memcheck over the replay and scorer tests (new cp.async rows, shared-atomic re-score masks)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for w in c1 c2 c3 c5; do timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log
for f in bench_c4 bench_ref bench_c1 bench_c2 bench_c3 bench_c5; do echo "== $f"; python - gpurun_out/$f.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), (d.get('parity') or {}).get('equal'), (d.get('roofline') or {}).get('frac'), d.get('clocks'), (d.get('stages') or {}).get('ms_serial_attribution'))
except Exception as e: print('ERR', e)
PY
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-python-reference --e2e-steps 1 > gpurun_out/ncu_launch_c4.log 2>&1
python tools/launch_table.py gpurun_out/launches_c4.csv > gpurun_out/launches_c4_table.txt 2>&1; head -12 gpurun_out/launches_c4_table.txt
SEL="tests/test_parity_gpu.py::test_small_cases tests/test_score_tc_gpu.py"
for tool in racecheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 --target-processes all \
    python -m pytest $SEL -q -x -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
