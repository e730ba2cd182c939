#!/bin/bash
# Mode L with all targets in the lowest bits (tile = bits 0..11, contiguous):
# bulk-copy producer (HQ_TC_LBULK=2) vs the cp.async kernel, on a dense state.
set -u
O=gpurun_out/lbulk; mkdir -p $O
HQ_TC_LBULK=2 timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -q --timeout 300 -p no:cacheprovider > $O/tests_lbulk2.log 2>&1; echo "tests rc=$?" >> $O/tests_lbulk2.log
P="low,b:0-1-2-3-4-6,b:0-1-2-3-5-6"
for r in 1 2; do
  timeout 600 python bench_sweep.py --reps 10 --ks 5,6 --placements "$P" > $O/cp_$r.jsonl 2>$O/cp_$r.err
  HQ_TC_LBULK=2 timeout 600 python bench_sweep.py --reps 10 --ks 5,6 --placements "$P" > $O/bulk_$r.jsonl 2>$O/bulk_$r.err
done
