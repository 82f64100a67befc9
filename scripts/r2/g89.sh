for d in 512 256 128 512 256; do echo "== mink $d"; KL_GEMM_PAIR_MINK=$d python scripts/r2/micro/gemm_c2.py; done
for i in 1 2; do for d in 512 256; do KL_GEMM_PAIR_MINK=$d timeout 600 python bench.py --config c2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 mink=$d', d['ms_per_step'])"; done; done
