for v in 0 3 2 -1; do
  MCB_K3_CTAS=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/k3_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/k3_$v.json').read().strip().splitlines()[-1]); c=d['config']
print('$v', round(d['value']/1e9,3), round(d['ms_per_step'],3), c.get('stage_ms_per_step'), c.get('stage_ms_serial_attribution',{}).get('k3_scorer'))"
done
