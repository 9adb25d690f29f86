# K3 -> ML replay pipeline depth sweep on C2 (MCB_ML_CHUNKS)
for v in 1 2 4 8; do
  MCB_ML_CHUNKS=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/chunk_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/chunk_$v.json').read().strip().splitlines()[-1]); c=d['config']
print('$v', round(d['value']/1e9,3), round(d['ms_per_step'],3), d['e2e']['value']/1e9, c.get('stage_ms_per_step'))"
done
