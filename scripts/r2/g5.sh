timeout 900 python scripts/r2/diag_model.py 2>&1 | tail -60
