nproc; python -c "import os; print(len(os.sched_getaffinity(0)))"
( time timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err ) 2>&1 | tail -3; echo ref rc $?
cat gpurun_out/r2_bench_ref.json
timeout 900 python bench.py --config c2 --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref_c2.json 2> gpurun_out/r2_bench_ref_c2.err; echo ref c2 rc $?
cat gpurun_out/r2_bench_ref_c2.json
