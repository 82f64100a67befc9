KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_new.so timeout 600 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -1
bash scripts/r2/ab_lib_bench.sh c4 2
bash scripts/r2/ab_lib_bench.sh c2 2
