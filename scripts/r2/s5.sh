TRACE=1 N=2 KL_HSP_CPL=24 timeout 60 python scripts/r2/micro/hsp512_time.py
TRACE=1 N=2 KL_HSP_CPL=1 timeout 60 python scripts/r2/micro/hsp512_time.py
