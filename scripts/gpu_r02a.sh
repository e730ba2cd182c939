#!/bin/bash
# Round 2, first GPU pass: smoke, the GPU test suite, a short bench (N=1)
# and the reference arm.  Everything goes to gpurun_out/r02a/.
set -u
OUT=gpurun_out/r02a
mkdir -p $OUT
nvidia-smi -L > $OUT/gpus.txt 2>&1; free -g >> $OUT/gpus.txt; nproc >> $OUT/gpus.txt
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.log 2>&1; echo "ref rc=$?" >> $OUT/bench_ref.log
timeout 600 python bench_sweep.py --reps 10 --ks 4,5,6 --placements low,spread,b:0-1-2-3-20-25,b:0-1-2-3-4,b:0-2-3-9-16,b:1-2-3-7-8-9,b:0-1-4-5-6 > $OUT/sweep32.log 2>&1; echo "sweep rc=$?" >> $OUT/sweep32.log
