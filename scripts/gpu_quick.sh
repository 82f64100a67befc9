# tests + bench + graph census (no ncu)
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "gdpa_fused" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'mfu', d['mfu']['value'], 'e2e', d['e2e']['value'])"
tail -3 gpurun_out/bench.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --op-census > /dev/null 2> gpurun_out/census.err; echo census rc $?
KL_PDL=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_nopdl.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_nopdl.json')); print('NO-PDL value', d['value'], 'ms', d['ms_per_step'])"
