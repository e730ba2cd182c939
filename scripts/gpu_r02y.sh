#!/bin/bash
# Is the k=6 mode-H pass energy-bound once the CTA imbalance is gone?  Diagnostic build of the
# tile-queue variant (scripts/r02_experiments/tile_queue.diff): diag 3 = no MMA, no conversion.
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02y
mkdir -p $OUT
L=paper_2111_06868_b200/lib/libhq_qdiag.so
for r in 1 2; do
for d in 3 0 1; do
  for st in 1 0; do
    HQ_LIB=$L HQ_TC_DIAG=$d HQ_TC_STATIC=$st timeout 300 python tools/power_probe.py --n 34 --reps 30 \
      --cases 6:b:8-9-10-20-21-22 > $OUT/d${d}_static${st}_$r.jsonl 2>> $OUT/err.log
  done
done
done
