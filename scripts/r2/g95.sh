timeout 600 python -m pytest tests/test_gpu_gemm_tc.py -q -x -k fold 2>&1 | tail -3
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -2
bash scripts/r2/ab_lib_bench.sh c4 3
bash scripts/r2/ab_lib_bench.sh c2 2
