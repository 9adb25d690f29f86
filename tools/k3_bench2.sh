bash tools/k3_bench.sh "$1"
python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c1 $1', d['value']/1e9, d['ms_per_step'], d['config']['stage_ms_serial_attribution']['k3_scorer'])"
python -m pytest tests/test_parity_gpu.py tests/test_smoke_gpu.py -q -x 2>&1 | tail -1
