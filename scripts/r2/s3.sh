python scripts/r2/micro/hsp512_time.py
JAG=1 python scripts/r2/micro/hsp512_time.py
N=1 timeout 300 ncu --set full -k regex:hsp_fwd512 -c 1 -o gpurun_out/hsp512_full python scripts/r2/micro/hsp512_time.py > gpurun_out/ncu_hsp.log 2>&1
