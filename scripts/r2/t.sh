timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "hsp" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_model_parity.py -q 2>&1 | tail -3
python scripts/r2/micro/hsp512_time.py
