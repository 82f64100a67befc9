KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_new.so timeout 600 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -2
for v in old new old new; do echo "== $v"; KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_$v.so python scripts/r2/micro/gemm_vs_cublas.py 2>&1 | head -8; done
bash scripts/r2/ab_lib_bench.sh c4 3
bash scripts/r2/ab_lib_bench.sh c2 2
