#!/bin/bash
# Mode-selection re-check after the mode-H low-target work (16-byte pattern
# pairs, swizzled 2-D TMA, lane-pair stores): is mode H now faster than mode L
# for the placements tc_use_mode_l still routes to L (bits 0 and 1 both
# targets, or three targets among bits 0..3)?
# 1) correctness of mode H on those placements (HQ_TC_MODE=H forces it);
# 2) same-box sweep, default routing vs forced H, two interleaved rounds.
set -u
O=gpurun_out/modesel; mkdir -p $O
HQ_TC_MODE=H timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -q --timeout 300 -p no:cacheprovider -k "low_targets or single_pass" > $O/tests_forceH.log 2>&1; echo "tests rc=$?" >> $O/tests_forceH.log
P6="low,b:0-1-10-20-21-22,b:0-1-2-15-20-25,b:1-2-3-12-20-28,b:0-2-3-9-17-30,b:0-1-8-9-10-11"
P5="low,b:0-1-12-20-28,b:1-2-3-15-25,b:0-2-3-9-30,b:0-1-2-3-20"
for r in 1 2; do
  timeout 600 python bench_sweep.py --reps 10 --ks 5,6 --placements "$P6,$P5" > $O/def_$r.jsonl 2>$O/def_$r.err
  HQ_TC_MODE=H timeout 600 python bench_sweep.py --reps 10 --ks 5,6 --placements "$P6,$P5" > $O/forceH_$r.jsonl 2>$O/forceH_$r.err
done
