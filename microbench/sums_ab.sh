#!/bin/bash
# A/B of the device-resident sums pre-pass: SKC_SUMS_BPS=0 is the previous k_build_sums,
# 4..8 the lean kernel at that many 256-thread blocks per SM (config 1, L2 flushed per step).
for v in 0 4 5 6 8 0 5; do
  echo "bps=$v $(SKC_SUMS_BPS=$v python microbench/build_overhead.py 2>&1 | grep flush=True)"
done
