timeout 600 python -m pytest tests/test_gpu_gemm_tc.py -q 2>&1 | tail -1
for nf in 0 1; do
KL_GEMM_NFAST=$nf timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_nf$nf.json 2> gpurun_out/r2_nf$nf.err; echo nf $nf rc $?
python scripts/r2/show.py gpurun_out/r2_nf$nf.json 2>&1 | head -3
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_nfauto.json 2> gpurun_out/r2_nfauto.err; echo auto rc $?
python scripts/r2/show.py gpurun_out/r2_nfauto.json 2>&1 | head -3
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_nfauto_c2.json 2> gpurun_out/r2_nfauto_c2.err; echo auto c2 rc $?
python scripts/r2/show.py gpurun_out/r2_nfauto_c2.json 2>&1 | head -2
