#!/bin/bash
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02h
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_pack.py tests/test_gpu_checked.py -q --timeout 800 -p no:cacheprovider > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log
cp gpurun_out/checked_run.log $OUT/ 2>/dev/null
timeout 900 python bench_sweep.py --reps 10 --ks 4,5,6 --placements low,spread,random0,b:0-1-2-3-20,b:0-1-4-5-6,b:0-1-2-9-12,b:0-2-3-9-16 > $OUT/sweep32.log 2>&1; echo "sweep rc=$?" >> $OUT/sweep32.log
python prof_one.py --n 32 --k 5 --placement low --reps 2 > $OUT/p_tcL5.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_tcL -s 1 -c 1 \
    -o $OUT/prof_tcL5 python prof_one.py --n 32 --k 5 --placement low --reps 2 > $OUT/ncu_tcL5.log 2>&1
echo "ncu rc=$?" >> $OUT/ncu_tcL5.log
