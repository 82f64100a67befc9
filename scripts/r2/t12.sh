KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_new.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_new.json 2> gpurun_out/b_new.err
python -c "import json; d=json.load(open('gpurun_out/b_new.json')); print('new', d['ms_per_step'])" 2>/dev/null || tail -1 gpurun_out/b_new.err
KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_new.so python scripts/r2/micro/hsp512_fb.py
KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_new.so timeout 300 python -m pytest tests -q -m gpu -k 'hsp or model_parity or grouped' 2>&1 | tail -1
