#!/bin/bash
# Full GPU validation + measurement pass (run under gpurun from the repo root).
# Writes everything to gpurun_out/.  Each ncu run follows the same command
# having exited 0 without ncu.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $OUT/clocks_bench.csv &
SMI=$!
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
kill $SMI
timeout 600 python bench.py --impl reference > $OUT/bench_ref.log 2>&1; echo "ref rc=$?" >> $OUT/bench_ref.log
timeout 900 python bench_sweep.py --reps 10 > $OUT/sweep32.log 2>&1; echo "sweep rc=$?" >> $OUT/sweep32.log
# launch list of the bench command (single metric, no replay)
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $OUT/plain_small.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_launches.log 2>&1
echo "launches rc=$?" >> $OUT/ncu_launches.log
# full capture of the tensor-core and SIMT kernels at 32q (same kernels as the bench)
python prof_one.py --n 32 --k 6 --placement b:8-9-10-20-21-22 --reps 2 > $OUT/p_tc.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_tcb -s 1 -c 1 \
    -o $OUT/prof_tc6 python prof_one.py --n 32 --k 6 --placement b:8-9-10-20-21-22 --reps 2 > $OUT/ncu_tc.log 2>&1
echo "ncu tc rc=$?" >> $OUT/ncu_tc.log
python prof_one.py --n 32 --k 6 --placement b:0-1-2-3-4-5 --reps 2 > $OUT/p_tcl.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_tcL -s 1 -c 1 \
    -o $OUT/prof_tcL6 python prof_one.py --n 32 --k 6 --placement b:0-1-2-3-4-5 --reps 2 > $OUT/ncu_tcl.log 2>&1
echo "ncu tcL rc=$?" >> $OUT/ncu_tcl.log
python prof_one.py --n 32 --k 4 --placement b:8-12-20-28 --reps 2 > $OUT/p_reg.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_reg -s 1 -c 1 \
    -o $OUT/prof_reg4 python prof_one.py --n 32 --k 4 --placement b:8-12-20-28 --reps 2 > $OUT/ncu_reg.log 2>&1
echo "ncu reg rc=$?" >> $OUT/ncu_reg.log
