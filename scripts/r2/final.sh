timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
python -c "import json; d=json.load(open('gpurun_out/final_c4.json')); print('c4', d['ms_per_step'], d['value'], d['mfu']['value'], d['e2e']['value'], d['clocks'], d['cpu_baseline']['value'])"
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' 2>&1 | tail -1
