#!/bin/bash
# Round 2 (session 2): power behaviour per pass type + fresh ncu --set full of the
# dominant kernel (the committed r02 prof_tc6 export was broken).
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02k
mkdir -p $OUT
timeout 600 python tools/power_probe.py --n 34 --reps 40 \
  --cases 1:b:20,2:b:3-20,3:b:8-20-28,6:b:16-17-18-22-23-24,6:b:8-9-10-20-21-22,5:b:16-17-18-22-23,4:b:8-12-20-28 \
  > $OUT/power34.jsonl 2> $OUT/power34.err; echo "power rc=$?" >> $OUT/power34.err
P="python prof_one.py --n 32 --k 6 --placement b:8-9-10-20-21-22 --reps 2"
$P > $OUT/p_tc6.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_tcb -s 1 -c 1 \
    -o $OUT/prof_tc6 $P > $OUT/ncu_tc6.log 2>&1
echo "ncu tc6 rc=$?" >> $OUT/ncu_tc6.log
ncu -i $OUT/prof_tc6.ncu-rep --page raw --csv > $OUT/prof_tc6_raw.csv 2>&1
ncu -i $OUT/prof_tc6.ncu-rep --page source --csv > $OUT/prof_tc6_source.csv 2>&1
ncu -i $OUT/prof_tc6.ncu-rep --page details --csv > $OUT/prof_tc6_details.csv 2>&1
