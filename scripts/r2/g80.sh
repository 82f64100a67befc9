timeout 600 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -2
for d in 0 1 0 1; do echo "== regs $d"; KL_GEMM_EPI_REGS=$d python scripts/r2/micro/gemm_vs_cublas.py 2>&1 | head -7; done
bash scripts/r2/ab_lib_bench.sh c4 3
