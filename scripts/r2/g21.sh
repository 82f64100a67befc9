timeout 300 python scripts/r2/diag_c1b.py 2>&1 | grep -E "lengths|ERR|ok"
