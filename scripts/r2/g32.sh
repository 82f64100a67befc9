KL_GEMM_TRACE=1 timeout 60 python scripts/r2/pair_check.py 2>&1 | tail -30
echo rc $?
