#!/bin/bash
# same-box A/B: dynamic tile queue (default) vs static split (HQ_TC_STATIC=1)
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02r
mkdir -p $OUT
C=6:b:8-9-10-20-21-22,5:b:16-17-18-22-23,6:b:0-1-2-3-4-5,5:b:0-1-2-3-4,4:b:0-1-2-3,6:b:0-7-13-20-26-33
for r in 1 2; do
  HQ_TC_STATIC=1 timeout 300 python tools/power_probe.py --n 34 --reps 30 --cases $C > $OUT/static_$r.jsonl 2>> $OUT/err.log
  timeout 300 python tools/power_probe.py --n 34 --reps 30 --cases $C > $OUT/dyn_$r.jsonl 2>> $OUT/err.log
done
HQ_TC_STATIC=1 timeout 300 python tools/pass_times.py > $OUT/pt_static.log 2>&1
timeout 300 python tools/pass_times.py > $OUT/pt_dyn.log 2>&1
