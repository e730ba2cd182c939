#!/bin/bash
# Same-box A/B of the layout cost model with the pair / swizzle kernels:
# HQ_LAYOUT_PAIR=0 (earlier weights) vs default, then the default bench line.
set -u
O=gpurun_out/lay; mkdir -p $O
for r in 1 2; do
  HQ_LAYOUT_PAIR=0 timeout 300 python tools/pass_times.py > $O/old_$r.jsonl 2>$O/old_$r.err
  timeout 300 python tools/pass_times.py > $O/new_$r.jsonl 2>$O/new_$r.err
done
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $O/clocks_bench.csv &
SMI=$!
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
kill $SMI
HQ_LAYOUT_PAIR=0 HQ_TC_SWZ=0 timeout 900 python bench.py --no-cpu-baseline > $O/bench_old.log 2>&1; echo "bench rc=$?" >> $O/bench_old.log
