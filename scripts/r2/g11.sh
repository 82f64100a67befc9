timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_c4.json 2> gpurun_out/r2_c4.err; echo rc $?
tail -3 gpurun_out/r2_c4.err
timeout 900 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_c2.json 2> gpurun_out/r2_c2.err; echo rc $?
python scripts/r2/show.py gpurun_out/r2_c4.json gpurun_out/r2_c2.json
