#!/bin/bash
# mode L paired converter stores: parity (TC tests) + same-box A/B against the previous build
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02x
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x --timeout 600 -p no:cacheprovider > $OUT/tc_tests.log 2>&1; echo "tests rc=$?" >> $OUT/tc_tests.log
C=6:b:0-1-2-3-4-5,5:b:0-1-2-3-4,4:b:0-1-2-3,6:b:1-2-3-4-5-6
for r in 1 2; do
  HQ_LIB=paper_2111_06868_b200/lib/libhq_base.so timeout 300 python tools/power_probe.py --n 34 --reps 30 --cases $C > $OUT/base_$r.jsonl 2>> $OUT/err.log
  timeout 300 python tools/power_probe.py --n 34 --reps 30 --cases $C > $OUT/new_$r.jsonl 2>> $OUT/err.log
done
