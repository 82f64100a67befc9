timeout 600 python -m pytest tests/test_gpu_ablations.py -q 2>&1 | grep -E "^E  |passed|failed" | cut -c1-300 | head -20
