timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for w in c2 c1; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['ms_per_step'], d['config']['stage_ms_per_step'], d['e2e']['value'])"; done
