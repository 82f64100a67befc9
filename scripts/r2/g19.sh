set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  |passed|failed" | cut -c1-300 | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for c in c4 c2 c1 c3; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err; echo $c rc $?
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_c4_full.json 2> gpurun_out/r2_bench_c4_full.err; echo full rc $?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo ref rc $?
python scripts/r2/show.py gpurun_out/r2_bench_c4_full.json gpurun_out/r2_bench_c2.json gpurun_out/r2_bench_c1.json gpurun_out/r2_bench_c3.json
cat gpurun_out/r2_bench_ref.json
