mkdir -p gpurun_out/ev
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/c4_launches_end.csv python bench.py --eager --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ev/ncu_launch_end.log 2>&1
python profiles/summarize_launches.py gpurun_out/ev/c4_launches_end.csv > gpurun_out/ev/c4_launches_end.txt
gzip -f gpurun_out/ev/c4_launches_end.csv
head -3 gpurun_out/ev/c4_launches_end.txt
