set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu --no-e2e --op-census > gpurun_out/c4_census.json 2> gpurun_out/c4_census.err; echo rc $?
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e --gemm-census > gpurun_out/c4_gemm.json 2> gpurun_out/c4_gemm.err; echo rc $?
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e --op-census > gpurun_out/c2_census.json 2> gpurun_out/c2_census.err; echo rc $?
