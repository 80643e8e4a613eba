#!/bin/bash
# A/B of the class-list windows' lockstep spread (SKC_LOCK_MB; 0 = off): builds one library
# per arm into gpurun_ab/lock_<MB>/ (here, before gpurun) and times config 1 / config 2 with
# each, plus dram bytes of k_build_cls from ncu.  usage: microbench/lock_ab.sh build|run
set -e
cd "$(dirname "$0")/.."
ARMS="${ARMS:-0 12 24 48}"
if [ "$1" = build ]; then
  for mb in $ARMS; do
    make -C paper_1506_04448_b200/csrc -j8 OUT=../../gpurun_ab/lock_$mb EXTRA=-DSKC_LOCK_MB=$mb ../../gpurun_ab/lock_$mb/libsketchcp_b200.so >/dev/null
  done
  exit 0
fi
mkdir -p gpurun_out
for mb in $ARMS; do
  for cfg in c2 c1; do
    echo -n "lock_mb=$mb " ; SKC_LIB_DIR=$PWD/gpurun_ab/lock_$mb python microbench/build_ab.py $cfg 10
  done
done
for mb in $ARMS; do
  SKC_LIB_DIR=$PWD/gpurun_ab/lock_$mb ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
     --clock-control none -k regex:k_build_cls --csv --log-file gpurun_out/lock_${mb}_c2.csv python microbench/build_once.py c2 2 > /dev/null 2>&1 || echo "ncu failed $mb"
  echo "lock_mb=$mb ncu:"; grep -E "k_build_cls" gpurun_out/lock_${mb}_c2.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | tail -8
done
