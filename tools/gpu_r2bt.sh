#!/bin/bash
# Multi-rank path on one box (2 gloo ranks sharing the GPU) + per-rank strong-scaling shares of C4 (--traces 4096/N)
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_c4_2ranks.json 2> gpurun_out/bench_c4_2ranks.err
tail -c 600 gpurun_out/bench_c4_2ranks.json; echo
for t in 2048 1024 512; do
timeout 600 python bench.py --traces $t --steps 5 --warmup 3 --no-cpu-baseline --no-python-reference --e2e-steps 1 > gpurun_out/share_$t.json 2>/dev/null
python - $t <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/share_{sys.argv[1]}.json').read().strip().splitlines()[-1])
print('traces', sys.argv[1], f"{d['value']:.3e}", round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages']['ms_serial_attribution'].items()}, d.get('parity',{}).get('equal'))
PY
done
