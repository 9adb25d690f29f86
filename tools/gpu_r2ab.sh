#!/bin/bash
# AR(1) hidden-state kernel: router tests, generator timing, C3 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_router_gpu.py tests/test_fullsize_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
python - <<'PY'
import torch, time
from paper_2601_17063_b200 import generator
for T in (65536, 1048576):
    generator.ar1_hidden(1024, 2048, 0.9, 1); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); H = generator.ar1_hidden(T, 2048, 0.9, 3); b.record(); b.synchronize()
    print(f"ar1_hidden T={T}: {a.elapsed_time(b):.2f} ms, {H.numel()*2/a.elapsed_time(b)/1e6:.0f} GB/s written")
PY
timeout 900 python bench.py --workload c3 --no-cpu-baseline --steps 3 --e2e-steps 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python -c "import json; d=json.loads(open('gpurun_out/bench_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['hit_rates'])"
