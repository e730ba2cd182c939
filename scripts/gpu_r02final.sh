#!/bin/bash
# Final validation of HEAD (fresh full build): smoke, GPU suite, bench, reference arm
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02final3
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
cp gpurun_out/checked_run.log gpurun_out/accuracy_320pass.json $OUT/ 2>/dev/null
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $OUT/clocks_bench.csv &
SMI=$!
timeout 1500 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
kill $SMI
timeout 900 python bench.py --impl reference > $OUT/bench_ref.log 2>&1; echo "ref rc=$?" >> $OUT/bench_ref.log
