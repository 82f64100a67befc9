timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "model_vs_oracle or hsp" 2>&1 | grep -E "^E  |passed|failed" | cut -c1-400 | head -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
