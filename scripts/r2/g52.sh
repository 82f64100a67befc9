mkdir -p gpurun_out
timeout 600 python scripts/r2/aten_sources.py c4 > gpurun_out/g52_c4.txt 2>&1; echo rc $?
timeout 600 python scripts/r2/aten_sources.py c3 > gpurun_out/g52_c3.txt 2>&1; echo rc $?
timeout 600 python scripts/r2/aten_sources.py c2 > gpurun_out/g52_c2.txt 2>&1; echo rc $?
