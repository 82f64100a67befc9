for v in f2fp pos f2fp pos; do cp scratch/lib_$v.so paper_2602_10016_b200/lib/libkunlun_sm100a.so; echo -n "$v: "; bash scripts/gpu_swa_quick.sh 2>&1 | grep "swa fwd"; done
