timeout 600 python -m pytest tests/test_gpu_branches.py -q -x 2>&1 | tail -2
for i in 1 2; do for c in 0 1; do KL_CLEAR_GRAD=$c timeout 600 python bench.py --config c3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 clear=$c', d['ms_per_step'])"; done; done
for i in 1 2; do for c in 0 1; do KL_CLEAR_GRAD=$c timeout 600 python bench.py --config c4 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 clear=$c', d['ms_per_step'])"; done; done
