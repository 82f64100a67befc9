nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/s1_pytest.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --op-census > gpurun_out/s1_census.json 2> gpurun_out/s1_census.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --gemm-census > gpurun_out/s1_gemm.json 2> gpurun_out/s1_gemm.err
