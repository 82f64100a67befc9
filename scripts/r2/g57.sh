mkdir -p gpurun_out
timeout 300 python scripts/r2/swa_time.py > /dev/null 2>&1; echo plain rc $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"swa_fwd_tc3|swa_bwd_dkv_tc3|swa_bwd_dq_tc3" -c 3 -o gpurun_out/swa3_c4 python scripts/r2/swa_time.py > gpurun_out/g57_ncu.log 2>&1; echo ncu rc $?
tail -3 gpurun_out/g57_ncu.log
