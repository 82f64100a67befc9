timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
python -c "import json; d=json.load(open('gpurun_out/b_c4.json')); print(d['ms_per_step'], d['value'], d['mfu']['value'], d['e2e']['value'])"
timeout 300 python scripts/r2/aten_sources.py c4 2>&1 | grep -v Warn | tail -14
