timeout 300 python scripts/r2/diag_c1.py c1 2>&1 | tail -35
