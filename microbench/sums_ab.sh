#!/bin/bash
# A/B of the lean sums pre-pass: fp32 loads in flight per lane and row (U) x resident blocks
# per SM. Builds one library per arm into gpurun_ab/sums_<U>_<MINB>/ (here, before gpurun).
# usage: microbench/sums_ab.sh build|run
set -e
cd "$(dirname "$0")/.."
ARMS="${ARMS:-4_5 8_5 8_4 8_3 4_6}"
if [ "$1" = build ]; then
  for a in $ARMS; do
    u=${a%_*}; m=${a#*_}
    make -C paper_1506_04448_b200/csrc -j8 OUT=../../gpurun_ab/sums_$a EXTRA="-DSKC_SUMS_U32=$u -DSKC_SUMS_MINB=$m" ../../gpurun_ab/sums_$a/libsketchcp_b200.so >/dev/null
  done
  exit 0
fi
for a in $ARMS; do
  echo -n "sums U_MINB=$a "; SKC_LIB_DIR=$PWD/gpurun_ab/sums_$a python microbench/build_ab.py c2 10
  SKC_LIB_DIR=$PWD/gpurun_ab/sums_$a ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_build_sums_lean -c 2 python microbench/build_once.py c2 2 2>&1 | grep -E "duration"
done
