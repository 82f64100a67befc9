timeout 120 python scripts/r2/prof_kernels.py all > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel|swa_bwd_dkv|swa_bwd_dq|swa_fwd_tc3" -s 4 -c 5 -o gpurun_out/r2_c4_kernels -f python scripts/r2/prof_kernels.py all > gpurun_out/ncu_r2.log 2>&1; echo ncu rc $?
tail -5 gpurun_out/ncu_r2.log
