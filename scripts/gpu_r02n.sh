#!/bin/bash
# Energy attribution of the k=6 mode-H pass under the power cap: diagnostic
# build (wrong results by design) with MMA / conversion / stores removed.
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02n
mkdir -p $OUT
for d in 0 1 2 4 3 5 6; do
  HQ_LIB=paper_2111_06868_b200/lib/libhq_diag.so HQ_TC_DIAG=$d timeout 300 python tools/power_probe.py --n 34 --reps 40 \
    --cases 6:b:8-9-10-20-21-22,5:b:16-17-18-22-23 > $OUT/diag$d.jsonl 2> $OUT/diag$d.err
  echo "diag $d rc=$?" >> $OUT/diag$d.err
done
