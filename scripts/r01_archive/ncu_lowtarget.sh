#!/bin/bash
# ncu --set full of apply_tcb at 32q with 0 / 1 targets in physical bits 0..3
# (the circuit's one-low-target k=6 passes run ~7% slower).
set -u
O=gpurun_out/lowt; mkdir -p $O
for pl in 8-9-10-20-21-22 1-8-9-10-20-21 0-8-9-10-20-21 3-8-9-10-20-21; do
  python prof_one.py --n 32 --k 6 --placement b:$pl --reps 2 > $O/p_$pl.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_tcb -s 1 -c 1 \
    -o $O/tc_$pl python prof_one.py --n 32 --k 6 --placement b:$pl --reps 2 > $O/ncu_$pl.log 2>&1
  echo "$pl rc=$?" >> $O/rc.log
  ncu -i $O/tc_$pl.ncu-rep --page raw --csv > $O/raw_$pl.csv 2>/dev/null
done
