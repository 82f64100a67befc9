timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu > gpurun_out/b_c4_$i.json 2> gpurun_out/b_c4_$i.err; python -c "import json; d=json.load(open('gpurun_out/b_c4_$i.json')); print('c4', d['ms_per_step'], d['value'], d['mfu']['value'], d['e2e']['value'])" 2>/dev/null || tail -1 gpurun_out/b_c4_$i.err; done
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' 2>&1 | tail -1
