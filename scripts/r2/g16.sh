timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "512_fused" 2>&1 | grep -E "^E  |passed|failed" | cut -c1-300 | head -20
