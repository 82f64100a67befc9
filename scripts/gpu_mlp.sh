for w in mlp mlp_noaux mlp_bias mlp_plain; do echo $w; timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_tc python scripts/probes/gemm_one.py $w 2>&1 | grep -E "duration" | tail -1; done
timeout 300 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'mfu', d['mfu']['value'], 'e2e', d['e2e']['value'])"
