#!/bin/bash
# A/B on one box: the K3-TC kernel of commit dea4ac9 vs HEAD (launch list, 512 traces).
mkdir -p gpurun_out
B="python bench.py --traces 512 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
L=paper_2601_17063_b200/lib/libmcb.so
cp $L /tmp/libmcb_new.so
for r in 1 2; do
for v in new old; do
  if [ $v = old ]; then cp gpurun_old/libmcb_old.so $L; else cp /tmp/libmcb_new.so $L; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_score_tc --csv --log-file gpurun_out/l_$v.csv $B > /dev/null 2>&1
  echo "$v"; python tools/launch_table.py gpurun_out/l_$v.csv | head -1
done; done
cp /tmp/libmcb_new.so $L
MCB_K3_GROUPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_score_tc --csv --log-file gpurun_out/l_v1.csv $B > /dev/null 2>&1
echo "variant 1"; python tools/launch_table.py gpurun_out/l_v1.csv | head -1
