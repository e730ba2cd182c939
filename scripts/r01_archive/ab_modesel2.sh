#!/bin/bash
# New mode-selection rule (tc_use_mode_l): full GPU tests, then a same-box
# sweep of the affected placements, new rule vs the earlier one
# (HQ_TC_MODESEL_V5=1), and the headline bench.
set -u
O=gpurun_out/modesel2; mkdir -p $O
python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/gputests.log 2>&1; echo "tests rc=$?" >> $O/gputests.log
P6="low,b:0-1-10-20-21-22,b:0-1-2-15-20-25,b:1-2-3-12-20-28,b:0-2-3-9-17-30,b:0-1-8-9-10-11"
P5="low,b:0-1-12-20-28,b:1-2-3-15-25,b:0-2-3-9-30,b:0-1-2-3-20"
for r in 1 2; do
  timeout 600 python bench_sweep.py --reps 10 --ks 5,6 --placements "$P6,$P5" > $O/new_$r.jsonl 2>$O/new_$r.err
  HQ_TC_MODESEL_V5=1 timeout 600 python bench_sweep.py --reps 10 --ks 5,6 --placements "$P6,$P5" > $O/old_$r.jsonl 2>$O/old_$r.err
done
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
