# launch list of one cfg3 batch (k_join kernels), then a full capture of the longest k_join_v launch
mkdir -p gpurun_out
PASSES=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_join" --csv python scripts/ncu_cfg3.py 2>/dev/null | grep -E "k_join" | awk -F'","' '{print $5, $(NF)}' | sed 's/"//g' | cat -n | sort -k3 -n -r | head -5
