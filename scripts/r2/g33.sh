KL_GEMM_TRACE=1 timeout 60 python scripts/r2/pair_check.py 2>&1 | grep -E "pair=|PASS|FAIL" | sort | uniq | head -20
for pr in 1 0; do KL_GEMM_PAIR=$pr timeout 120 python scripts/r2/gemm_time.py 2>&1 | sed "s/^/pair$pr /"; done
