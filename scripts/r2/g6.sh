timeout 900 python scripts/r2/diag_model.py 2>&1 | grep -A2 "1024, 32" | head -12
timeout 600 python -m pytest tests/test_gpu_model_parity.py -q -s 2>&1 | grep -E "worst|^E  |passed|failed" | cut -c1-600
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "gdpa_vs_oracle or model_vs_oracle or mask_bitexact" 2>&1 | grep -E "^E  |passed|failed" | cut -c1-400 | head -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
