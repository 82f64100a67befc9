timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |passed|failed" | cut -c1-400 | head -30
