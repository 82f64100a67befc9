mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_model_parity.py -q > gpurun_out/g48_tests.log 2>&1; echo tests rc $?
tail -30 gpurun_out/g48_tests.log
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu --no-e2e --gemm-census > gpurun_out/g48_c3.json 2> gpurun_out/g48_c3.err; echo c3 rc $?
grep "^gemm" gpurun_out/g48_c3.err | head -40
