#!/bin/bash
# k=6 mode H sustained at 32q vs 34q (is the 34q gap a size effect?), k=1 for reference
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02o
mkdir -p $OUT
for n in 32 33 34; do
  timeout 300 python tools/power_probe.py --n $n --reps 60 --cases 1:b:20,6:b:8-9-10-20-21-22,5:b:16-17-18-22-23 > $OUT/n$n.jsonl 2> $OUT/n$n.err
  HQ_LIB=paper_2111_06868_b200/lib/libhq_diag.so HQ_TC_DIAG=3 timeout 300 python tools/power_probe.py --n $n --reps 60 --cases 6:b:8-9-10-20-21-22 > $OUT/n${n}_diag3.jsonl 2>> $OUT/n$n.err
done
