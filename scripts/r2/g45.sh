timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "gdpa" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_model_parity.py -q -k "d512" 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_c4.json 2> gpurun_out/r2_c4.err; echo rc $?
python scripts/r2/show.py gpurun_out/r2_c4.json 2>&1 | head -14
