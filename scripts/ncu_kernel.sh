#!/bin/bash
# usage: scripts/ncu_kernel.sh REGEX COUNT OUTDIR  -- full ncu capture of matching kernels in one
# cfg2 batch (scripts/ncu_target.py), summarised per source line into OUTDIR (small text files)
mkdir -p "$3"
SLICE=${SLICE:-100} timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$1" -c "$2" -o /tmp/prof_k python scripts/ncu_target.py > "$3/ncu.log" 2>&1
python scripts/ncu_lines.py /tmp/prof_k.ncu-rep "$3/l" "$2"
ncu -i /tmp/prof_k.ncu-rep --page details --csv > "$3/details.csv" 2>/dev/null
