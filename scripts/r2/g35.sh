for c in c2 c4; do for pr in 0 1; do
KL_GEMM_PAIR=$pr timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab_$c$pr.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ab_$c$pr.json')); t=d['roofline_table']['gemm']; print('$c pair=$pr', round(d['ms_per_step'],3), 'gemm ms', round(t['ms_per_step'],3))"
done; done
