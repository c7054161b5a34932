bash scripts/profile_r02c.sh r02i
bash scripts/bench_all.sh r02i
