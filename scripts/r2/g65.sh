for i in 1 2; do
for v in NONE KL_AB_GIOLD KL_AB_STK; do
env $v=1 timeout 600 python bench.py --config c2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'])"
done
env KL_AB_GIOLD=1 KL_AB_OLDSTK=1 timeout 600 python bench.py --config c2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('GIOLD+catrows', d['ms_per_step'])"
done
