mkdir -p gpurun_out/ev
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"swa_bwd|swa_rowdot" -s 3 -c 3 -o gpurun_out/ev/c4_swab -f python scripts/r2/prof_kernels.py swa > gpurun_out/ev/ncu_swab.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gdpa_fwd512|gdpa_bwd512" -s 2 -c 2 -o gpurun_out/ev/c4_gdpa -f python scripts/r2/prof_kernels.py gdpa > gpurun_out/ev/ncu_gdpa.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel" -c 12 -o gpurun_out/ev/c4_wide -f python scripts/r2/micro/gemm_wide.py > gpurun_out/ev/ncu_wide.log 2>&1
python profiles/summarize_ncu.py gpurun_out/ev/c4_swab.ncu-rep gpurun_out/ev/c4_gdpa.ncu-rep gpurun_out/ev/c4_wide.ncu-rep > gpurun_out/ev/ncu_c4_kernels2.txt 2>&1
python profiles/make_ncu_json.py gpurun_out/ev/ncu_c4_B32_b.json gpurun_out/ev/c4_swab.ncu-rep gpurun_out/ev/c4_gdpa.ncu-rep > /dev/null 2>&1
ls gpurun_out/ev
