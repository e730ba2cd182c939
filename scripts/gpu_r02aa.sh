#!/bin/bash
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02aa
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench_dm.py --N 15 --steps 3 > $OUT/bench_dm.log 2>&1; echo "dm rc=$?" >> $OUT/bench_dm.log
timeout 600 python bench_dm.py --N 15 --steps 3 --fuse c7 > $OUT/bench_dm_c7.log 2>&1; echo "dm rc=$?" >> $OUT/bench_dm_c7.log
