for v in old new; do
KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_$v.json 2> gpurun_out/b_$v.err
echo $v rc $?; python -c "import json; d=json.load(open('gpurun_out/b_$v.json')); print('$v', d['ms_per_step'])" 2>/dev/null || tail -1 gpurun_out/b_$v.err
done
