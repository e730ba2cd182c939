#!/bin/bash
# same-box A/B: HEAD library (static split, no queue warp) vs working tree (tile queue)
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02s
mkdir -p $OUT
C=6:b:8-9-10-20-21-22,5:b:16-17-18-22-23,6:b:0-1-2-3-4-5,5:b:0-1-2-3-4,4:b:0-1-2-3
for r in 1 2; do
  HQ_LIB=paper_2111_06868_b200/lib/libhq_head.so timeout 300 python tools/power_probe.py --n 34 --reps 30 --cases $C > $OUT/head_$r.jsonl 2>> $OUT/err.log
  timeout 300 python tools/power_probe.py --n 34 --reps 30 --cases $C > $OUT/dyn_$r.jsonl 2>> $OUT/err.log
done
