timeout 900 ncu --set full --clock-control none --import-source on -k regex:swa_.*tc3 -c 3 -o gpurun_out/swa3_full -f python scripts/probes/swa_tc_probe.py bwd_only 128 1024 4 128 0 full > gpurun_out/ncu_swa3.log 2>&1; echo ncu rc $?
tail -2 gpurun_out/ncu_swa3.log
