timeout 300 python -m pytest tests/test_gpu_gemm_tc.py -q -x -k "arow" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -2
for d in 1 0 1 0; do echo "== arow $d"; KL_GEMM_AROW=$d python scripts/r2/micro/gemm_vs_cublas.py 2>&1 | head -5; done
