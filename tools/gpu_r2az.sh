#!/bin/bash
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "next_use" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_next_use --csv --log-file gpurun_out/l_nu.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/l_nu.csv | head -3
timeout 900 python bench.py --no-cpu-baseline --steps 5 --e2e-steps 2 > gpurun_out/b.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],1), d['e2e']['ms_per_step'], d['stages']['ms_serial_attribution'])"
