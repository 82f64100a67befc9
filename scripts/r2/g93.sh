timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
bash scripts/r2/ab_lib_bench.sh c4 3
bash scripts/r2/ab_lib_bench.sh c2 3
bash scripts/r2/ab_lib_bench.sh c3 1
