timeout 300 python scripts/r2/swa_trace.py
