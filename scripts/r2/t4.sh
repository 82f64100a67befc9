python scripts/r2/micro/gemm_vs_cublas.py 2>&1 | head -5
KL_GEMM_WIDE_ALL=1 python scripts/r2/micro/gemm_vs_cublas.py 2>&1 | head -5
