#!/bin/bash
# Block planner (hq_fuse_blocks, 34q d20 k<=6: 37 passes): tests, smoke, bench.
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02l
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $OUT/clocks_bench.csv &
SMI=$!
timeout 1200 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
kill $SMI
timeout 600 python tools/pass_times.py > $OUT/pass_times.log 2>&1; echo "pt rc=$?" >> $OUT/pass_times.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
