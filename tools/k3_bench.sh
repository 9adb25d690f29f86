# one C2 bench line: value, ms/step, K3 alone (serial attribution)
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('${1:-run}', d['value']/1e9, d['ms_per_step'], d['config']['stage_ms_serial_attribution']['k3_scorer'], d['scorer_uncertain_events'])"
