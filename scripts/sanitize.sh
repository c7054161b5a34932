#!/bin/bash
# compute-sanitizer evidence: memcheck, racecheck, synccheck, initcheck on the small workload.
R=${1:-r02}
mkdir -p gpurun_out/profiles
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python scripts/sanitize_target.py > gpurun_out/profiles/${R}_sanitizer_$tool.txt 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/profiles/${R}_sanitizer_summary.txt
  tail -3 gpurun_out/profiles/${R}_sanitizer_$tool.txt | tee -a gpurun_out/profiles/${R}_sanitizer_summary.txt
done
