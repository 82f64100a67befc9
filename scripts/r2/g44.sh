timeout 120 python scripts/r2/prof_kernels.py gdpa > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gdpa_fwd512|gdpa_bwd512|gemm_tc" -s 4 -c 6 -o gpurun_out/r2_c4_gdpa -f python scripts/r2/prof_kernels.py gdpa > gpurun_out/ncu_r2c.log 2>&1; echo ncu rc $?
timeout 120 python scripts/r2/prof_kernels.py swa > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"swa_" -s 5 -c 5 -o gpurun_out/r2_c4_swa -f python scripts/r2/prof_kernels.py swa > gpurun_out/ncu_r2d.log 2>&1; echo ncu rc $?
