for st in 8 2 3 4 8; do echo "== stages<=$st"; KL_GEMM_STAGES=$st python scripts/r2/micro/gemm_c2.py; KL_GEMM_STAGES=$st python scripts/r2/micro/gemm_vs_cublas.py 2>&1 | head -3; done
