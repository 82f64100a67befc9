# usage: bash scripts/r2/ab_lib_bench.sh <config> [rounds]: bench.py with lib/ab_old.so vs lib/ab_new.so, alternating
C=$1; N=${2:-2}
for i in $(seq $N); do
for v in old new; do
  KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_$v.so timeout 600 python bench.py --config $C --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'])"
done; done
