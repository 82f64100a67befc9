mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/g54_tests.log 2>&1; echo tests rc $?
tail -3 gpurun_out/g54_tests.log
for c in c4 c3 c2; do
timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/g54_$c.json 2> gpurun_out/g54_$c.err; echo $c rc $?
done
