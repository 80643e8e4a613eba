#!/bin/bash
# A/B of the dense build: the experiment library (SKC_LIB_DIR=$1) against the in-tree one,
# alternating arms, each in its own process: bash microbench/ab_build.sh <dir> [configs] [rounds]
dir=$1; cfgs=${2:-"c2 c1"}; rounds=${3:-2}
for c in $cfgs; do for r in $(seq $rounds); do
 SKC_LIB_DIR=$dir python microbench/build_ab.py $c 20 2>&1 | tail -1 | sed "s/^/A $c: /"
 python microbench/build_ab.py $c 20 2>&1 | tail -1 | sed "s/^/B $c: /"
done; done
