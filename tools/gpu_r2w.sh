#!/bin/bash
# K3-TC weight-block order: per-K-block streaming (HEAD) vs part-major (gpurun_old): precision + timing.
mkdir -p gpurun_out
B="python bench.py --traces 512 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
L=paper_2601_17063_b200/lib/libmcb.so
cp $L /tmp/libmcb_new.so
for v in new old; do
  if [ $v = old ]; then cp gpurun_old/libmcb_old.so $L; else cp /tmp/libmcb_new.so $L; fi
  timeout 600 python -m pytest tests/test_score_tc_gpu.py -q -s -p no:cacheprovider -k "calibrated or equal_float64_ranks" 2>&1 | grep "normwise\|E=64, 3\|passed\|failed"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_score_tc --csv --log-file gpurun_out/l_$v.csv $B > /dev/null 2>&1
  echo "$v"; python tools/launch_table.py gpurun_out/l_$v.csv | head -1
done
cp /tmp/libmcb_new.so $L
