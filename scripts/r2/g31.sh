for bn in auto 128 64; do
  if [ $bn = auto ]; then timeout 120 python scripts/r2/gemm_time.py; else KL_GEMM_BN=$bn timeout 120 python scripts/r2/gemm_time.py; fi
done 2>&1 | grep TF
