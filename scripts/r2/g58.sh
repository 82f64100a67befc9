mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/g58_tests.log 2>&1; echo tests rc $?
tail -3 gpurun_out/g58_tests.log
timeout 600 python scripts/r2/aten_sources.py c4 > gpurun_out/g58_aten_c4.txt 2>&1; echo rc $?
for c in c4 c3 c2; do
timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/g58_$c.json 2> gpurun_out/g58_$c.err; echo $c rc $?
done
