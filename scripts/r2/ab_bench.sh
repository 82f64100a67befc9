# usage: bash scripts/r2/ab_bench.sh <config> [rounds]: bench.py of ab/old vs the current tree, alternating
C=$1; N=${2:-3}
for i in $(seq $N); do
  (cd ab/old && timeout 600 python bench.py --config $C --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', d['ms_per_step'])")
  timeout 600 python bench.py --config $C --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', d['ms_per_step'])"
done
