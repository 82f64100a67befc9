timeout 300 python -m pytest tests/test_gpu_gemm_tc.py tests/test_gpu_branches.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
KL_GEMM_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --eager > /dev/null 2> gpurun_out/trace.err; echo rc $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'mfu', d['mfu']['value'], 'e2e', d['e2e']['value'])"
tail -3 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --eager > gpurun_out/ncu_launch.log 2>&1; echo ncu rc $?
