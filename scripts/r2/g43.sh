timeout 120 python scripts/r2/prof_kernels.py all > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel|swa_fwd_tc3|swa_bwd_dkv_tc3|swa_bwd_dq_tc3|gdpa_fwd512|gdpa_bwd512|hsp_fwd512|hsp_bwd512|adam_kernel" -s 9 -c 9 -o gpurun_out/r2_c4_full -f python scripts/r2/prof_kernels.py all > gpurun_out/ncu_r2b.log 2>&1; echo ncu rc $?
tail -3 gpurun_out/ncu_r2b.log
