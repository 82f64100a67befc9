KL_GEMM_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --eager > /dev/null 2> gpurun_out/trace.err; echo rc $?
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "gi or model" 2>&1 | tail -2
