for nf in 0 1; do
KL_GEMM_NFAST=$nf timeout 120 python scripts/r2/prof_kernels.py gemm > /dev/null 2>&1 && \
KL_GEMM_NFAST=$nf timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_tc_kernel -s 1 -c 1 python scripts/r2/prof_kernels.py gemm 2>&1 | grep -E "gpu__time|dram__bytes|hit_rate|tensor_cycles" 
done
