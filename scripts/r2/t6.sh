timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python bench.py --eager --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
python profiles/summarize_launches.py gpurun_out/c4_launches.csv > gpurun_out/c4_launches.txt
head -45 gpurun_out/c4_launches.txt
