KL_HSP_DBG=1 TRACE=1 N=2 KL_HSP_CPL=24 timeout 60 python scripts/r2/micro/hsp512_time.py 2>&1 | head -8
N=1 timeout 300 ncu --set full -k regex:hsp_fwd512s -c 1 -o gpurun_out/hsp512s_full python scripts/r2/micro/hsp512_time.py > gpurun_out/ncu_hsp.log 2>&1
