run() { env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_k.json 2> gpurun_out/b_k.err; python -c "import json; d=json.load(open('gpurun_out/b_k.json')); print('$*', d['ms_per_step'])" 2>/dev/null || echo "$* failed"; }
run X=0
run KL_GEMM_WIDE_K=1024
run KL_GEMM_WIDE_K=256
run KL_GEMM_RWIDE_KB=16
run KL_GEMM_RWIDE_KB=2
run X=0
run KL_GEMM_WIDE_K=1024
