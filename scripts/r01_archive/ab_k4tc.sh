#!/bin/bash
# k = 4 on the tensor cores (mode H, HQ_TC_K4=1) vs the SIMT FFMA2 kernel:
# correctness of the whole GPU suite with the switch on, then a same-box
# sweep of k = 4 at placements without low targets (and the default ones).
set -u
O=gpurun_out/k4tc; mkdir -p $O
HQ_TC_K4=1 timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/gputests_k4.log 2>&1; echo "tests rc=$?" >> $O/gputests_k4.log
P="low,high,spread,random0,random1,random2,b:4-9-17-25,b:5-6-20-30,b:8-12-20-28,b:10-11-12-13,b:7-15-22-31"
for r in 1 2; do
  timeout 600 python bench_sweep.py --reps 10 --ks 4 --placements "$P" > $O/simt_$r.jsonl 2>$O/simt_$r.err
  HQ_TC_K4=1 timeout 600 python bench_sweep.py --reps 10 --ks 4 --placements "$P" > $O/tc_$r.jsonl 2>$O/tc_$r.err
done
