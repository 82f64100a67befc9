timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "dtype1" 2>&1 | grep -E "^E  |passed|failed" | cut -c1-400 | head -60
