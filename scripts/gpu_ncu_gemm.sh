for w in qkv dx; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/gemm_$w -f python scripts/probes/gemm_one.py $w > gpurun_out/ncu_gemm_$w.log 2>&1; echo ncu $w rc $?
done
