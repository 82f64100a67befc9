KL_GEMM_NOWIDE=1 python scripts/r2/micro/gemm_wide.py 2>&1 | grep "x256x"
python scripts/r2/micro/gemm_wide.py 2>&1 | grep "x256x"
timeout 300 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -1
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
python -c "import json; d=json.load(open('gpurun_out/b_c2.json')); print('c2', d['ms_per_step'], d['value'], d['mfu']['value'])"
