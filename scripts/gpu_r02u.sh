#!/bin/bash
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02u
mkdir -p $OUT
timeout 1200 python bench.py --no-cpu-baseline --sweep-reps 0 --e2e-steps 0 --steps 3 --warmup 3 > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
