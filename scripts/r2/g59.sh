bash scripts/r2/ab_bench.sh c2 3
bash scripts/r2/ab_bench.sh c4 2
