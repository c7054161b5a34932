bash scripts/profile_r02c.sh r02g
bash scripts/bench_all.sh r02g
