#!/bin/bash
# Round 2, third GPU pass: tensor-core and pack tests, the sweep cells the
# mode-L and k=4 work targets, an ncu capture of the new mode-L kernel, bench.
set -u
OUT=gpurun_out/r02c
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_pack.py tests/test_gpu_tc.py tests/test_gpu_accuracy.py -q --timeout 600 -p no:cacheprovider > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log
cp gpurun_out/accuracy_*.json $OUT/ 2>/dev/null
timeout 600 python bench_sweep.py --reps 10 --ks 4,5,6 --placements low,spread,random0,b:0-1-2-3-20-25,b:0-1-2-3-4,b:0-2-3-9-16,b:1-2-3-7-8-9,b:0-1-4-5-6 > $OUT/sweep32.log 2>&1; echo "sweep rc=$?" >> $OUT/sweep32.log
python prof_one.py --n 32 --k 6 --placement low --reps 2 > $OUT/p_tcl.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_tcL -s 1 -c 1 \
    -o $OUT/prof_tcL6 python prof_one.py --n 32 --k 6 --placement low --reps 2 > $OUT/ncu_tcl.log 2>&1
echo "ncu tcL rc=$?" >> $OUT/ncu_tcl.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
