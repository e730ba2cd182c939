#!/bin/bash
# Round 2, second GPU pass: apply+pack tests, the full GPU suite, the
# compute-sanitizer runs, and one ncu --set full capture of the FP16 mode-L
# kernel.  Everything goes to gpurun_out/r02b/.
set -u
OUT=gpurun_out/r02b
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_pack.py -x -q --timeout 600 -p no:cacheprovider > $OUT/packtests.log 2>&1; echo "pack tests rc=$?" >> $OUT/packtests.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
python tools/sanitize_run.py > $OUT/sanitize_plain.log 2>&1; echo "plain rc=$?" >> $OUT/sanitize_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitize_$tool.log
done
python prof_one.py --n 32 --k 6 --placement low --reps 2 > $OUT/p_tcl.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_tcL -s 1 -c 1 \
    -o $OUT/prof_tcL6_fp16 python prof_one.py --n 32 --k 6 --placement low --reps 2 > $OUT/ncu_tcl.log 2>&1
echo "ncu tcL rc=$?" >> $OUT/ncu_tcl.log
