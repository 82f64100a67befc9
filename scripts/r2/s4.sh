OLD=1 timeout 60 python scripts/r2/micro/hsp512_time.py
timeout 60 python scripts/r2/micro/hsp512_time.py
JAG=1 timeout 60 python scripts/r2/micro/hsp512_time.py
KL_HSP_CPL=7 JAG=1 timeout 60 python scripts/r2/micro/hsp512_time.py
KL_HSP_CPL=5 timeout 60 python scripts/r2/micro/hsp512_time.py
