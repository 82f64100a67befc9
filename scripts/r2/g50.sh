mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/g50_tests.log 2>&1; echo tests rc $?
tail -5 gpurun_out/g50_tests.log
timeout 900 python bench.py --config c3 --no-cpu > gpurun_out/g50_c3.json 2> gpurun_out/g50_c3.err; echo c3 rc $?
