#!/bin/bash
# mode L energy attribution (experiment builds, wrong results by design): LEXP 1 no epilogue
# stores, 2 no converter shared stores, 4 no MMAs, 3 = 1 + 2
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02w
mkdir -p $OUT
C=6:b:0-1-2-3-4-5,5:b:0-1-2-3-4
for v in base 1 2 4 3 base; do
  if [ $v = base ]; then L=paper_2111_06868_b200/lib/libhq.so; else L=paper_2111_06868_b200/lib/libhq_lexp$v.so; fi
  HQ_LIB=$L timeout 300 python tools/power_probe.py --n 34 --reps 30 --cases $C >> $OUT/lexp_$v.jsonl 2>> $OUT/err.log
done
