# C2 segment length / warm-up sweep (MCB_SEG_EV / MCB_SEG_NW)
for cfg in "0 0" "256 128" "256 64" "128 64" "128 32"; do
  set -- $cfg
  MCB_SEG_EV=$1 MCB_SEG_NW=$2 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print('$1/$2', round(d['value']/1e9,3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in c['stage_ms_serial_attribution'].items()}, d['segmented_replay'])"
done
