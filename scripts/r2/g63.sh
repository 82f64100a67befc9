for i in 1 2; do
env KL_AB_HSPDO=1 KL_AB_DQZ=1 KL_AB_GI=1 KL_AB_ROWS=1 KL_AB_ZERO=1 KL_LIB_PATH=$PWD/ab/old/paper_2602_10016_b200/lib/libkunlun_sm100a.so timeout 600 python bench.py --config c2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ALL+oldlib', d['ms_per_step'])"
env KL_AB_HSPDO=1 KL_AB_DQZ=1 KL_AB_GI=1 KL_AB_ROWS=1 KL_AB_ZERO=1 timeout 600 python bench.py --config c2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ALL', d['ms_per_step'])"
(cd ab/old && timeout 600 python bench.py --config c2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', d['ms_per_step'])")
(cd ab/old && KL_LIB_PATH=/root/repo/paper_2602_10016_b200/lib/libkunlun_sm100a.so timeout 600 python bench.py --config c2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old+newlib', d['ms_per_step'])")
done
