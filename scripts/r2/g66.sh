timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_model_parity.py tests/test_gpu_grouped.py -q -x > gpurun_out/g66_tests.log 2>&1; echo tests rc $?
tail -2 gpurun_out/g66_tests.log
bash scripts/r2/ab_bench.sh c2 2
bash scripts/r2/ab_bench.sh c4 1
