timeout 600 python -m pytest tests/test_gpu_trainer.py tests/test_gpu_ablations.py -q -x 2>&1 | grep -E "^E  |passed|failed|Error" | cut -c1-300 | head -20
