timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "hsp" 2>&1 | grep -E "^E  |passed|failed" | cut -c1-300 | head -20
timeout 900 python -m pytest tests/test_gpu_model_parity.py -q -s 2>&1 | grep -E "worst|^E  |passed|failed" | cut -c1-400 | head -20
