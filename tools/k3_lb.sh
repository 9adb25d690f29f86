python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lb4', d['value']/1e9, d['ms_per_step'], d['config']['stage_ms_serial_attribution']['k3_scorer'])"
sed -i 's/TE ? 4 : 1/TE ? 3 : 1/' paper_2601_17063_b200/csrc/mcb_kernels.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lb3', d['value']/1e9, d['ms_per_step'], d['config']['stage_ms_serial_attribution']['k3_scorer'])"
