#!/bin/bash
# validation of the block-planner state: bench (default), reference arm, ncu launch list
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02v
mkdir -p $OUT
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $OUT/clocks_bench.csv &
SMI=$!
timeout 1500 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
kill $SMI
timeout 900 python bench.py --impl reference > $OUT/bench_ref.log 2>&1; echo "ref rc=$?" >> $OUT/bench_ref.log
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --sweep-reps 0 --no-other-configs"
$B > $OUT/plain_small.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/launches.csv $B > $OUT/ncu_launches.log 2>&1
echo "launches rc=$?" >> $OUT/ncu_launches.log
