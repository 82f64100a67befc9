bash scripts/r2/ab_bench.sh c2 3
