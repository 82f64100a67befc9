mkdir -p gpurun_out
bash scripts/r2/ab.sh scripts/r2/swa_time.py > gpurun_out/g56_ab.txt 2>&1
cat gpurun_out/g56_ab.txt
