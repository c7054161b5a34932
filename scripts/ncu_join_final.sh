#!/bin/bash
# ncu capture of the final (largest) join step of one cfg2 batch: k_join_v launches only
mkdir -p gpurun_out/lines3
SLICE=100 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_join_v|k_join_seg" -c 12 -o /tmp/prof3 python scripts/ncu_target.py > gpurun_out/ncu3.log 2>&1
python scripts/ncu_lines.py /tmp/prof3.ncu-rep gpurun_out/lines3/l 12
ncu -i /tmp/prof3.ncu-rep --page details --csv > gpurun_out/lines3/details.csv 2>/dev/null
