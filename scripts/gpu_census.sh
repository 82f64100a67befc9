timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --gemm-census > /dev/null 2> gpurun_out/gemm_census.err; echo gemm census rc $?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --op-census > /dev/null 2> gpurun_out/op_census.err; echo op census rc $?
