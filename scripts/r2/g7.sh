timeout 600 python -m pytest tests/test_gpu_model_parity.py -q -s 2>&1 | grep -E "worst|^E  |passed|failed" | cut -c1-600
timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | grep -E "^E  |passed|failed" | cut -c1-400 | head -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
