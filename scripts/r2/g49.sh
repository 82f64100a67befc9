mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/g49_tests.log 2>&1; echo tests rc $?
tail -5 gpurun_out/g49_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g49_smoke.log 2>&1; echo smoke rc $?
tail -3 gpurun_out/g49_smoke.log
for c in c1 c2 c3; do
timeout 900 python bench.py --config $c > gpurun_out/g49_$c.json 2> gpurun_out/g49_$c.err; echo $c rc $?
done
timeout 900 python bench.py > gpurun_out/g49_c4.json 2> gpurun_out/g49_c4.err; echo c4 rc $?
