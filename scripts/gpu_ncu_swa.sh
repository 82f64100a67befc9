timeout 300 python tests/swa_tc_probe.py bwd_only 128 1024 4 128 0 full > gpurun_out/swa_probe.log 2>&1; echo probe rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:swa_.*tc2 -c 3 -o gpurun_out/swa_full -f python tests/swa_tc_probe.py bwd_only 128 1024 4 128 0 full > gpurun_out/ncu_swa.log 2>&1; echo ncu rc $?
tail -3 gpurun_out/ncu_swa.log
