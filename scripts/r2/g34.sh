timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | grep -E "^E  |passed|failed" | cut -c1-300 | head -20
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_c4.json 2> gpurun_out/r2_c4.err; echo rc $?
python scripts/r2/show.py gpurun_out/r2_c4.json 2>&1 | head -4
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_c2.json 2> gpurun_out/r2_c2.err; echo rc $?
python scripts/r2/show.py gpurun_out/r2_c2.json 2>&1 | head -3
