for d in 0 1 0 1; do echo "== dbg $d"; KL_GEMM_DBG_EPI=$d python scripts/r2/micro/gemm_vs_cublas.py 2>&1 | head -2; done
