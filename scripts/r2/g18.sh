timeout 600 python -m pytest tests/test_gpu_refbind.py tests/test_gpu_dist_model.py -q -x 2>&1 | grep -E "^E  |passed|failed|Error" | cut -c1-300 | head -20
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "numerics" 2>&1 | grep -E "^E  |passed|failed|Error" | cut -c1-300 | head -20
