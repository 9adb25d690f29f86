# C1 (E = 128, 2,048 tokens) segment sweep: MCB_SEG_EV / MCB_SEG_NW / MCB_SEG_PASSES
for cfg in "0 0 0" "512 128 0" "512 256 0" "1024 256 0" "256 128 0" "512 128 1" "-1 0 0"; do
  set -- $cfg
  MCB_SEG_EV=$1 MCB_SEG_NW=$2 MCB_SEG_PASSES=$3 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print('$1/$2/$3', round(d['value']/1e9,3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in c['stage_ms_per_step'].items() if k!='note'}, d['segmented_replay']['fixup_events'])"
done
