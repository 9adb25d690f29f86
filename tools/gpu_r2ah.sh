#!/bin/bash
# Round-2 evidence refresh: smoke, every workload's bench line, the reference arm (C4).
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
for w in c1 c2 c3; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
done
timeout 1500 python bench.py --workload c5 --steps 2 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
for w in c4 c1 c2 c3 c5 ref; do python - $w <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/bench_{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], f"{d['value']:.3e}", round(d['ms_per_step'],2), f"e2e {d['e2e']['value']:.3e}", 'parity', (d.get('parity') or {}).get('equal'), 'roof', d.get('roofline',{}) and round(d['roofline']['frac'],4))
PY
done
