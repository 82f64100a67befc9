timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_c4.json 2> gpurun_out/r2_c4.err; echo rc $?
python scripts/r2/show.py gpurun_out/r2_c4.json
