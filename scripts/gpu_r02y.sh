bash scripts/profile_r02c.sh r02c
bash scripts/bench_all.sh r02c
