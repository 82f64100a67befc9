timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "swa" 2>&1 | tail -2
timeout 120 python scripts/probes/swa_tc_probe.py fwd 8 1024 4 128 0 full 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:swa_ python scripts/probes/swa_tc_probe.py bwd_only 128 1024 4 128 0 full 2>&1 | grep -E "swa_|duration" | head -12
