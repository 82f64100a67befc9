timeout 120 python scripts/r2/swa_wide.py 2>&1 | tail -6
