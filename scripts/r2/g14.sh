timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --gemm-census > /dev/null 2> gpurun_out/c4_gemm2.err; echo rc $?
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --op-census > /dev/null 2> gpurun_out/c4_census2.err; echo rc $?
grep "^gemm" gpurun_out/c4_gemm2.err | head -45 | cut -c1-200
sed -n '/by kernel/,/by call site/p' gpurun_out/c4_census2.err | head -40 | cut -c1-160
