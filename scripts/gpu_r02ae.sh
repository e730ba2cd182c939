#!/bin/bash
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02ae
mkdir -p $OUT
timeout 900 python tools/cublas_baseline.py --n 31 --reps 5 > $OUT/cublas.jsonl 2> $OUT/err.log; echo "rc=$?" >> $OUT/err.log
