KL_GEMM_TRACE=1 python scripts/r2/micro/gemm_wide.py 2>&1 | grep -E "wide|gemm_tc M=1536" | head -12
KL_GEMM_NOWIDE=1 python scripts/r2/micro/gemm_wide.py
timeout 600 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -2
