bash scripts/r2/ab.sh scripts/r2/swa_time.py
