#!/bin/bash
# tile queue (dynamic tile scheduling) in the tensor-core kernels
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02q2
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x --timeout 600 -p no:cacheprovider > $OUT/tc_tests.log 2>&1; echo "tests rc=$?" >> $OUT/tc_tests.log
timeout 300 python tools/power_probe.py --n 34 --reps 40 --cases 6:b:8-9-10-20-21-22,5:b:16-17-18-22-23,6:b:0-1-2-3-4-5,5:b:0-1-2-3-4 > $OUT/power34.jsonl 2> $OUT/power34.err
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $OUT/clocks_bench.csv &
SMI=$!
timeout 1200 python bench.py --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
kill $SMI
