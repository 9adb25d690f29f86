# C2 segment length / warm-up sweep under the replays-after-K3 schedule
for cfg in ${CFGS:-"0 0" "384 192" "384 256" "768 256" "1024 256" "512 320"}; do
  set -- $cfg
  MCB_SEG_EV=$1 MCB_SEG_NW=$2 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']; print('$1/$2', round(d['value']/1e9,3), round(d['ms_per_step'],3), {k: round(v,3) for k,v in c['stage_ms_per_step'].items() if k!='note'}, d['segmented_replay']['fixup_events'])"
done
