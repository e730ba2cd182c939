#!/bin/bash
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02z
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
cp gpurun_out/checked_run.log $OUT/ 2>/dev/null
