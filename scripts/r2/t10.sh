timeout 300 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
python -c "import json; d=json.load(open('gpurun_out/b_c4.json')); print(d['ms_per_step'], d['value'], d['mfu']['value'], d['e2e']['value'])"
KL_GEMM_NOWIDE_R=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_c4b.json 2> gpurun_out/b_c4b.err
python -c "import json; d=json.load(open('gpurun_out/b_c4b.json')); print('nowide_r', d['ms_per_step'])"
