mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "swa or window or mha" > gpurun_out/g51_tests.log 2>&1; echo tests rc $?
tail -3 gpurun_out/g51_tests.log
timeout 900 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_model_parity.py -q > gpurun_out/g51_tests2.log 2>&1; echo tests2 rc $?
tail -3 gpurun_out/g51_tests2.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/g51_c4.json 2> gpurun_out/g51_c4.err; echo c4 rc $?
timeout 900 python bench.py --config c3 --no-cpu --no-e2e > gpurun_out/g51_c3.json 2> gpurun_out/g51_c3.err; echo c3 rc $?
