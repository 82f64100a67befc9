KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_trace.so timeout 300 python scripts/r2/swa_trace_fwd.py
