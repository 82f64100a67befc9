# tile-order A/B: GEMM tests, per-shape ncu durations with / without KL_GEMM_M_FAST, full GPU tests, bench
timeout 300 python -m pytest tests/test_gpu_gemm_tc.py -q -x 2>&1 | tail -2
for w in qkv bias mlp_noaux; do for mf in 0 1; do
if [ $mf = 1 ]; then export KL_GEMM_M_FAST=1; else unset KL_GEMM_M_FAST; fi
echo -n "$w mfast=$mf "; timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_tc python scripts/probes/gemm_one.py $w 2>&1 | grep -E "duration|dram" | tail -2 | tr '\n' ' '; echo
done; done
unset KL_GEMM_M_FAST
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_nf.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_nf.json')); print('nfast ms', d['ms_per_step'])"
KL_GEMM_M_FAST=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_mf.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_mf.json')); print('mfast ms', d['ms_per_step'])"
done
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench rc $?
python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'mfu', d['mfu']['value'], 'e2e', d['e2e']['value'])"
