timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --op-census > /dev/null 2> gpurun_out/census.err; echo census rc $?
