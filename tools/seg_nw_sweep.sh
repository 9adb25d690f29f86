# C2 warm-up sweep at the default segment length (MCB_SEG_NW)
for nw in 0 192 128 64; do
  MCB_SEG_NW=$nw python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print('nw=$nw', round(d['value']/1e9,3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in c['stage_ms_serial_attribution'].items()}, d['segmented_replay'])"
done
