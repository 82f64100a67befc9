for pen in 2000 8000 20000 2000 8000 20000; do
KL_GEMM_WS_PENALTY=$pen timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_p.json 2> gpurun_out/b_p.err
python -c "import json; d=json.load(open('gpurun_out/b_p.json')); print('pen $pen', d['ms_per_step'])" 2>/dev/null || tail -1 gpurun_out/b_p.err
done
