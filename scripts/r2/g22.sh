timeout 300 python scripts/r2/diag_swa.py 2>&1 | tail
