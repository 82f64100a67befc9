mkdir -p gpurun_out
timeout 300 python scripts/r2/swa_time.py > gpurun_out/g55_swa.txt 2>&1; echo rc $?
cat gpurun_out/g55_swa.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "swa or window or mha" > gpurun_out/g55_tests.log 2>&1; echo tests rc $?
tail -2 gpurun_out/g55_tests.log
