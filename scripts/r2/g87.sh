python scripts/r2/micro/gemm_c2.py
echo "== BN=128"; KL_GEMM_BN=128 python scripts/r2/micro/gemm_c2.py
echo "== NFAST=1"; KL_GEMM_NFAST=1 python scripts/r2/micro/gemm_c2.py
echo "== EPI1"; KL_GEMM_EPI1=1 python scripts/r2/micro/gemm_c2.py
