set -e
for c in c1 c2; do for f in 0 1 0 1; do SKC_CLS_FLAT=$f python microbench/build_ab.py $c 10; done; done
