for d in 0 1 2 0 1 2; do echo "== dbg $d"; KL_GEMM_DBG_EPI=$d python scripts/r2/micro/gemm_c2.py; done
