#!/bin/bash
# NLOW / NLOW_MAXC sweep for K4-wide lowest-keys victims (edits the box's scratch copy and rebuilds)
mkdir -p gpurun_out
run() {
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; return; }
  for a in "--policies lfu,belady" "--workload c5 --steps 2"; do
  timeout 600 python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline --no-python-reference --e2e-steps 1 > gpurun_out/pol.json 2>/dev/null
  python - "$1 $a" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/pol.json').read().strip().splitlines()[-1])
print(sys.argv[1], f"{d['value']:.3e}", round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages']['ms_serial_attribution'].items()})
PY
  done
}
F=paper_2601_17063_b200/csrc/mcb_wide.cu
for cfg in "4 32" "6 32" "2 32" "4 48"; do
  set -- $cfg
  sed -i -E "s/constexpr int NLOW = [0-9]+;/constexpr int NLOW = $1;/; s/constexpr uint32_t NLOW_MAXC = [0-9]+;/constexpr uint32_t NLOW_MAXC = $2;/" $F
  grep -n "constexpr int NLOW\|NLOW_MAXC =" $F | head -2
  run "NLOW=$1 MAXC=$2"
done
