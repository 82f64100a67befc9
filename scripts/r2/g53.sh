mkdir -p gpurun_out
timeout 600 python scripts/r2/aten_sources.py c4 > gpurun_out/g53_c4.txt 2>&1; echo rc $?
