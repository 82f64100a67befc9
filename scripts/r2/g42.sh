timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "arbitrary_mask or jagged" 2>&1 | grep -E "^E  |passed|failed|Error" | cut -c1-300 | head -20
