#!/bin/bash
# Correctness of the swizzled-TMA apply_tcb (GPU tests), then a same-box A/B of
# HQ_TC_SWZ=0/1 on the 34q bench circuit (pass_times, interleaved) and the 32q sweep at k=5,6.
set -u
O=gpurun_out/swz2; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > $O/gputests.log 2>&1; echo "tests rc=$?" >> $O/gputests.log
for r in 1 2; do
  HQ_TC_SWZ=0 timeout 300 python tools/pass_times.py > $O/base_$r.jsonl 2>$O/base_$r.err
  timeout 300 python tools/pass_times.py > $O/swz_$r.jsonl 2>$O/swz_$r.err
done
HQ_TC_SWZ=0 timeout 600 python bench_sweep.py --reps 10 --ks 5,6 > $O/sw_base.jsonl 2>&1
timeout 600 python bench_sweep.py --reps 10 --ks 5,6 > $O/sw_swz.jsonl 2>&1
