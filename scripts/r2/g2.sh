set -x
timeout 600 python -m pytest tests/test_gpu_model_parity.py -x -q -s 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "gdpa_vs_oracle or mask_bitexact or hsp_vs_oracle or model_vs_oracle" 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
