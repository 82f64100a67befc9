timeout 600 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -3
python scripts/r2/micro/gemm_vs_cublas.py 2>&1 | head -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
python -c "import json; d=json.load(open('gpurun_out/b_c4.json')); print(d['ms_per_step'], d['value'], d['mfu']['value'], d['e2e']['value'])"
