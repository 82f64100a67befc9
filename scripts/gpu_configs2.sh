# the other BASELINE configs (c1 tiny, c3 8-layer CompSkip 16 events, c4 d=512 T=4096) + c2 again, 10 timed steps
for c in c1 c3 c4 c2; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc $?
python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', 'value', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'mfu', round(d['mfu']['value'],4), 'e2e', round(d['e2e']['value'],1))" 2>&1 | tail -1
tail -1 gpurun_out/bench_$c.err
done
