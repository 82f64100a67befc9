for f in 3 1; do KL_GEMM_FOLD=$f CFG=c4 timeout 600 python scripts/r2/diag_c3_gemm.py 2>/dev/null | grep -v Warn > gpurun_out/fold_$f.txt; done
