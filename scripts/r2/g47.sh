mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_model_parity.py -x -q > gpurun_out/g47_tests.log 2>&1; echo tests rc $?
tail -30 gpurun_out/g47_tests.log
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/g47_c3.json 2> gpurun_out/g47_c3.err; echo c3 rc $?
tail -5 gpurun_out/g47_c3.err
