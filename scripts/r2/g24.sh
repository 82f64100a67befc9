for bn in auto 64 96 128 192 256; do
  if [ $bn = auto ]; then timeout 120 python scripts/r2/diag_gemm2.py; else KL_GEMM_BN=$bn timeout 120 python scripts/r2/diag_gemm2.py; fi
done 2>&1 | grep BN
