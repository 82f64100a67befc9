# usage: bash scripts/r2/ab.sh <script> [args]: runs the script with lib/ab_old.so and lib/ab_new.so alternately (3 rounds)
for i in 1 2 3; do
for v in old new; do
echo "== $v"; KL_LIB_PATH=$PWD/paper_2602_10016_b200/lib/ab_$v.so timeout 600 python "$@"
done; done
