timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "gdpa" 2>&1 | grep -E "^E  |passed|failed" | cut -c1-300 | head -20
timeout 900 python -m pytest tests/test_gpu_model_parity.py -q -s 2>&1 | grep -E "worst|^E  |passed|failed" | cut -c1-400 | head -20
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_c4.json 2> gpurun_out/r2_c4.err; echo rc $?
python scripts/r2/show.py gpurun_out/r2_c4.json
