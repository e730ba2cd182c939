#!/bin/bash
# same-box A/B: HEAD (static split) vs tile queue for mode H + single epilogue multiply,
# and the same build with the static split (HQ_TC_STATIC=1)
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02ab
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x --timeout 600 -p no:cacheprovider > $OUT/tc_tests.log 2>&1; echo "tests rc=$?" >> $OUT/tc_tests.log
C=6:b:8-9-10-20-21-22,6:b:16-17-18-22-23-24,5:b:16-17-18-22-23,6:b:0-1-2-3-4-5
for r in 1 2; do
  HQ_LIB=paper_2111_06868_b200/lib/libhq_base.so timeout 300 python tools/power_probe.py --n 34 --reps 30 --cases $C > $OUT/base_$r.jsonl 2>> $OUT/err.log
  timeout 300 python tools/power_probe.py --n 34 --reps 30 --cases $C > $OUT/new_$r.jsonl 2>> $OUT/err.log
  HQ_TC_STATIC=1 timeout 300 python tools/power_probe.py --n 34 --reps 30 --cases $C > $OUT/newstatic_$r.jsonl 2>> $OUT/err.log
done
HQ_LIB=paper_2111_06868_b200/lib/libhq_base.so timeout 300 python tools/pass_times.py > $OUT/pt_base.log 2>&1
timeout 300 python tools/pass_times.py > $OUT/pt_new.log 2>&1
