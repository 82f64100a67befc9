# end-of-session evidence: every config's bench line, smoke
for c in c1 c2 c3; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/final_$c.json 2> gpurun_out/final_$c.err; python -c "import json; d=json.load(open('gpurun_out/final_$c.json')); print('$c', d['ms_per_step'], d['value'], d.get('mfu',{}).get('value'), d['e2e']['value'])" || tail -3 gpurun_out/final_$c.err; done
timeout 900 python bench.py > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
python -c "import json; d=json.load(open('gpurun_out/final_c4.json')); print('c4', d['ms_per_step'], d['value'], d['mfu']['value'], d['e2e']['value'], d['clocks'], d['cpu_baseline']['value'])"
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' 2>&1 | tail -1
