bash scripts/r2/ab.sh scripts/r2/gemm_dw_time.py 2>&1 | head -8
