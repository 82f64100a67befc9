for i in 1 2; do
for v in NONE KL_AB_HSPDO KL_AB_DQZ; do
env $v=1 timeout 600 python bench.py --config c2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'])"
done; done
env KL_AB_HSPDO=1 KL_AB_DQZ=1 KL_AB_GI=1 KL_AB_ROWS=1 KL_AB_ZERO=1 timeout 600 python bench.py --config c2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ALL', d['ms_per_step'])"
(cd ab/old && timeout 600 python bench.py --config c2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', d['ms_per_step'])")
