#!/bin/bash
# (Record only: these hooks were removed after this A/B showed no gain.)
# A/B of the class-list kernel's end-of-window hooks (config 1, L2 flushed per step):
# SKC_CLS_TAIL_ROWS / SKC_CLS_TAIL_CHUNK (shorter grabs near a window's end) and
# SKC_CLS_MIGRATE_MIN (no migration to windows with at most that many rows left).
run() { echo "$1 | $(env $1 python microbench/build_overhead.py 2>&1 | grep flush=True)"; }
run "X=0"
run "SKC_CLS_TAIL_ROWS=4096 SKC_CLS_TAIL_CHUNK=8"
run "SKC_CLS_TAIL_ROWS=8192 SKC_CLS_TAIL_CHUNK=8"
run "SKC_CLS_TAIL_ROWS=8192 SKC_CLS_TAIL_CHUNK=16"
run "SKC_CLS_TAIL_ROWS=16384 SKC_CLS_TAIL_CHUNK=16"
run "SKC_CLS_MIGRATE_MIN=512"
run "SKC_CLS_MIGRATE_MIN=2048"
run "SKC_CLS_MIGRATE_MIN=8192"
run "SKC_CLS_TAIL_ROWS=8192 SKC_CLS_TAIL_CHUNK=8 SKC_CLS_MIGRATE_MIN=2048"
run "X=0"
