#!/bin/bash
# launch list of the host path with 8 upload pieces (1,024 traces) vs 1
for u in 8 1; do
MCB_UPLOAD_PIECES=$u timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_up$u.csv python tools/e2e_probe.py 1024 > /dev/null 2>&1
echo "== pieces $u"; python tools/launch_table.py gpurun_out/l_up$u.csv | grep -v "at::" | head -12
done
