./scripts/r2/micro/tmem_bw
python scripts/r2/micro/gemm_vs_cublas.py
