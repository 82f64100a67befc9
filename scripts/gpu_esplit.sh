# split-epilogue A/B: GEMM tests, per-shape ncu durations with / without KL_GEMM_NO_ESPLIT, full GPU tests, bench
timeout 300 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -2
for w in qkv dx res bias mlp_noaux; do for ns in 0 1; do
if [ $ns = 1 ]; then export KL_GEMM_NO_ESPLIT=1; else unset KL_GEMM_NO_ESPLIT; fi
echo -n "$w nosplit=$ns "; timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_tc python scripts/probes/gemm_one.py $w 2>&1 | grep -E "duration" | tail -1
done; done
unset KL_GEMM_NO_ESPLIT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench rc $?
python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'mfu', d['mfu']['value'], 'e2e', d['e2e']['value'])"
KL_GEMM_NO_ESPLIT=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_nosplit.json 2>/dev/null; echo nosplit rc $?
python -c "import json; d=json.load(open('gpurun_out/bench_nosplit.json')); print('nosplit value', d['value'], 'ms', d['ms_per_step'])"
