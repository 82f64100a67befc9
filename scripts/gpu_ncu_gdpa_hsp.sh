# ncu --set full of one launch each of the fused GDPA and HSP kernels inside the c2 training step
# (eager mode so kernels are launched individually; numbers summarised into profiles/r1_gdpa_hsp_ncu.txt)
for k in gdpa_fwd gdpa_bwd hsp_fwd hsp_bwd; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -c 1 -o gpurun_out/$k -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --eager > gpurun_out/ncu_$k.log 2>&1; echo ncu $k rc $?
tail -2 gpurun_out/ncu_$k.log
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --gemm-census > /dev/null 2> gpurun_out/gemm_census.err; echo gemm census rc $?
timeout 600 python scripts/torch_glue_census.py > gpurun_out/glue_census.txt 2>&1; echo glue census rc $?
