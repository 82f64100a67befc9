# round-2 evidence: bench lines (c4 headline with CPU baseline + reference arm, c1-c3), launch list, ncu --set full of the hot kernels
mkdir -p gpurun_out/ev
timeout 900 python bench.py > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev/bench_ref_c4.json 2> gpurun_out/ev/bench_ref_c4.err
for c in c1 c2 c3; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/ev/bench_$c.json 2> gpurun_out/ev/bench_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/c4_launches.csv python bench.py --eager --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ev/ncu_launch.log 2>&1
python profiles/summarize_launches.py gpurun_out/ev/c4_launches.csv > gpurun_out/ev/c4_launches.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel|swa_fwd_tc3|swa_bwd_dkv_tc3|swa_bwd_dq_tc3|gdpa_fwd512|gdpa_bwd512|hsp_fwd512|hsp_bwd512|adam_kernel" -s 9 -c 9 -o gpurun_out/ev/c4_full -f python scripts/r2/prof_kernels.py all > gpurun_out/ev/ncu_full.log 2>&1
python profiles/summarize_ncu.py gpurun_out/ev/c4_full.ncu-rep > gpurun_out/ev/ncu_c4_kernels.txt 2>&1
python profiles/make_ncu_json.py gpurun_out/ev/ncu_c4_B32.json gpurun_out/ev/c4_full.ncu-rep > /dev/null 2>&1
ls -la gpurun_out/ev
