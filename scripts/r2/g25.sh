timeout 600 python -m pytest tests/test_gpu_gemm_tc.py -q 2>&1 | tail -2
timeout 300 python scripts/r2/diag_c1.py c1 2>&1 | tail -3
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_bench_c1.json 2> gpurun_out/r2_bench_c1.err; echo c1 rc $?
python scripts/r2/show.py gpurun_out/r2_bench_c1.json | head -3
