timeout 300 env KL_SMOKE_VERBOSE=1 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -12
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gdpa_vs_oracle and 4-256-16-1024 and dtype1" 2>&1 | grep -E "Error|assert|^E" | head -20
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "model_vs_oracle and False-dtype1" 2>&1 | grep -E "Error|assert|^E" | head -20
