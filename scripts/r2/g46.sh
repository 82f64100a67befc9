timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --eager > gpurun_out/launch_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c4_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --eager > gpurun_out/ncu_launch.log 2>&1; echo ncu rc $?
ls -la gpurun_out/r2_c4_launches.csv
