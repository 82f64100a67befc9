for c in c1 c3 c4; do
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc $?
python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', 'value', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'mfu', round(d['mfu']['value'],4))" 2>&1 | tail -1
tail -2 gpurun_out/bench_$c.err
done
