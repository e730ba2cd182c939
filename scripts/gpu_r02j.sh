#!/bin/bash
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02j
mkdir -p $OUT
timeout 900 python bench_sweep.py --reps 10 --ks 4,5 --placements low,spread,random0,random1,b:8-12-20-28,b:0-1-2-3 > $OUT/sweep32.log 2>&1; echo "sweep rc=$?" >> $OUT/sweep32.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config 34q --kmax 4 --fuse c7 > $OUT/bench_k4.log 2>&1; echo "bench rc=$?" >> $OUT/bench_k4.log
