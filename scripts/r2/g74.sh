KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_new.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "swa or window or mha" 2>&1 | tail -1
bash scripts/r2/ab.sh scripts/r2/swa_time.py 2>&1 | head -6
