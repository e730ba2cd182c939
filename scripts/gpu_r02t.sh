#!/bin/bash
# planner (LOOK 4/6 best-of-two, 36 passes): smoke, GPU suite, bench, pass times
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02t
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $OUT/clocks_bench.csv &
SMI=$!
timeout 1200 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
kill $SMI
timeout 600 python tools/pass_times.py > $OUT/pass_times.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
cp gpurun_out/accuracy_320pass.json gpurun_out/checked_run.log $OUT/ 2>/dev/null
