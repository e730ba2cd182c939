#!/bin/bash
# Round 2 validation + measurement pass (one B200).  Every ncu command runs
# after the same command exited 0 without ncu.  Output: gpurun_out/r02g/.
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02g
mkdir -p $OUT
nvidia-smi -q -d CLOCK,POWER > $OUT/smi_before.txt 2>&1
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
cp gpurun_out/accuracy_320pass.json gpurun_out/checked_run.log $OUT/ 2>/dev/null
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $OUT/clocks_bench.csv &
SMI=$!
timeout 1200 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
kill $SMI
timeout 900 python bench.py --impl reference > $OUT/bench_ref.log 2>&1; echo "ref rc=$?" >> $OUT/bench_ref.log
timeout 900 python tools/remap_timeline.py --n 30 --G 8 > $OUT/timeline30_G8.json 2> $OUT/timeline.err
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --sweep-reps 0"
$B > $OUT/plain_small.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/launches.csv $B > $OUT/ncu_launches.log 2>&1
echo "launches rc=$?" >> $OUT/ncu_launches.log
for spec in "6 b:8-9-10-20-21-22 apply_tcb tc6" "5 spread apply_tcb tc5" "6 low apply_tcL tcL6" "5 low apply_tcL tcL5" "4 b:8-12-20-28 apply_reg reg4"; do
  set -- $spec
  python prof_one.py --n 32 --k $1 --placement $2 --reps 2 > $OUT/p_$4.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
      -o $OUT/prof_$4 python prof_one.py --n 32 --k $1 --placement $2 --reps 2 > $OUT/ncu_$4.log 2>&1
  echo "ncu $4 rc=$?" >> $OUT/ncu_$4.log
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second
for pl in spread low; do
  python tools/sweep_ncu.py 32 $pl > $OUT/pk_$pl.log 2>&1 && \
    timeout 900 ncu --metrics $M --clock-control none --csv --log-file $OUT/ncu_per_k_${pl}32.csv python tools/sweep_ncu.py 32 $pl > $OUT/ncu_pk_$pl.log 2>&1
  echo "per-k $pl rc=$?" >> $OUT/ncu_pk_$pl.log
done
timeout 1500 python tools/oracle_full.py --n 30 --cycles 20 --seed 1000 > $OUT/oracle_full_30q.json 2>&1
timeout 300 python tools/oracle_full.py --n 12 --cycles 10 --seed 0 --threads 1 > $OUT/oracle_full_12q_1thread.json 2>&1
