# non-ML replay during K3 (1) or after it next to the ML replay (0), C2 and C1
for o in 0 1; do
  for w in c2 c1; do
    MCB_OVERLAP=$o python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('overlap=$o $w', round(d['value']/1e9,3), round(d['ms_per_step'],3), d['e2e']['value']/1e9, {k: round(v,3) for k,v in d['config']['stage_ms_per_step'].items() if k!='note'})"
  done
done
