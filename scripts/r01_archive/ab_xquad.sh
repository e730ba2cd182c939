#!/bin/bash
# GPU tests with xpair on every bit-0-free pass, then same-box A/B HQ_TC_XQUAD=0 vs default
# (pass_times, 34q circuit), the default bench line, and the k = 5, 6 sweep.
set -u
O=gpurun_out/xq; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > $O/gputests.log 2>&1; echo "tests rc=$?" >> $O/gputests.log
for r in 1 2; do
  HQ_TC_XQUAD=0 timeout 300 python tools/pass_times.py > $O/old_$r.jsonl 2>$O/old_$r.err
  timeout 300 python tools/pass_times.py > $O/new_$r.jsonl 2>$O/new_$r.err
done
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $O/clocks_bench.csv &
SMI=$!
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
kill $SMI
timeout 600 python bench_sweep.py --reps 10 --ks 5,6 > $O/sweep.jsonl 2>&1
