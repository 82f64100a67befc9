timeout 300 python scripts/r2/diag_gemm.py 2>&1 | tail -20
