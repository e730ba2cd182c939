#!/bin/bash
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02e
mkdir -p $OUT
timeout 900 python bench_sweep.py --reps 10 --ks 3,4,5,6 --placements low,spread,random0,random1,b:0-1-2-3-20-25,b:0-2-3-9-16,b:1-2-3-7-8-9,b:0-1-4-5-6 > $OUT/sweep32.log 2>&1; echo "sweep rc=$?" >> $OUT/sweep32.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 800 -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
