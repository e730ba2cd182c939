#!/bin/bash
# Same-box A/B: swizzled 2-D TMA on every apply_tcb pass (HQ_TC_SWZ=2) vs default.
set -u
O=gpurun_out/swzall; mkdir -p $O
for r in 1 2; do
  timeout 300 python tools/pass_times.py > $O/def_$r.jsonl 2>$O/def_$r.err
  HQ_TC_SWZ=2 timeout 300 python tools/pass_times.py > $O/all_$r.jsonl 2>$O/all_$r.err
done
