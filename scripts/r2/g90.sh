for d in 0 1 0 1; do echo "== krot $d"; KL_GEMM_KROT=$d python scripts/r2/micro/gemm_c2.py; KL_GEMM_KROT=$d python scripts/r2/micro/gemm_vs_cublas.py 2>&1 | head -7; done
