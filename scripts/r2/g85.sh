timeout 900 python -m pytest tests -q -m gpu -x -k "hsp or grouped or model_parity or pool or pma" 2>&1 | tail -2
for i in 1 2; do for v in old new; do echo "== $v"; KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_$v.so SHAPE=128,1024,256,160 python scripts/r2/micro/hsp_fb.py; done; done
bash scripts/r2/ab_lib_bench.sh c2 3
bash scripts/r2/ab_lib_bench.sh c3 2
