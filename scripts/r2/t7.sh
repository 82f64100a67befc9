timeout 300 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -2
python scripts/r2/micro/gemm_vs_cublas.py 2>&1 | head -5
KL_GEMM_WIDE_K=512 python scripts/r2/micro/gemm_vs_cublas.py 2>&1 | head -5
KL_GEMM_WIDE_K=512 timeout 300 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -2
